"""CPU oracle for the Varuna pipeline executor — TEST INFRASTRUCTURE ONLY.

Everything under ``oracle/`` is a checker. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. The product package
(``paper_2111_04007_b200``) never imports it and has no CPU fallback.

Contents (each function cites the reference file:line it restates; paths are
relative to /root/reference, ``sp/`` = ``pkg/src/spotpipe/``):

* ``schedule``  — Varuna rule-simulation plan + GPipe plan + zero-delay replay
  (sp/scheduler.py:88-97, 128-284, 307-373).
* ``engine``    — the opportunistic replica event kernel, ``run_replica``
  (sp/engine/py_kernel.py:41-360).
* ``partition`` — ``assign_stages`` / ``identify_cutpoints`` / ``memory_check``
  (sp/partitioner.py:109-436).
* ``gpt2_fp32`` — fp32 PyTorch-CPU GPT-2 stage model and a sequential pipeline
  executor that walks the Varuna schedule (F no-save, R from stash, B), the
  loss/gradient oracle. The reference has no tensor math (SPEC.md:18,
  79-80), so THIS PART IS PARITY-UNPINNED against the reference: it is
  pinned only against its own single-process, non-pipelined forward/backward.
* ``gen_golden`` — runs the reference (spotpipe 0.1.0) in the build
  container and writes ``tests/golden/*.json``; the control-plane oracle
  above is pinned against those fixtures by ``tests/test_oracle_golden.py``.
"""
