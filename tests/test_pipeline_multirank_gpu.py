"""The multi-rank data plane — IPC-mapped activation/gradient rings, the
interprocess-event + shm handshake, the gradient put kernel, the DP (C1),
pipeline-wide norm/overflow (C2) and tied-embedding (C3) collectives,
opportunistic dispatch, re-tuning and plan-driven morphing — against the
fp32 CPU oracle, as 2 or 4 processes.

Every case runs on ONE B200 (all ranks on cuda:0, CUDA IPC between the
processes, gloo collectives: NCCL refuses duplicate GPUs) so the
single-GPU ``pytest -m gpu`` covers it; the ``multigpu`` variants run the
same checks one GPU per rank over NCCL when the box has the GPUs.

Tolerances as tests/test_pipeline_gpu.py: loss |Δ|/|loss| <= 5e-3,
per-tensor gradient relative L2 <= 3e-2 (dist_pipeline_check.py)."""

import re

import pytest
import torch

from tests._dist import launch

pytestmark = pytest.mark.gpu

PIPE_CASES = [
    # (nproc, P, D, config, extra args)
    (2, 2, 1, "tiny", []),
    (4, 2, 2, "tiny", []),
    (4, 4, 1, "tiny", []),
    (4, 2, 2, "tiny_bert", []),
    (2, 2, 1, "tiny_ragged", []),
    # M_total = 27 at m=4, N=4, D=2: replica 1 gets 11 rows — one partial and
    # one empty micro-batch; the loss is the mean over 27 samples
    (4, 2, 2, "tiny", ["--global-batch", "27"]),
    # K7 dropout-recompute across stages and replicas: F on stage 0 and R
    # before B regenerate the same masks; replicas draw different ones
    (4, 2, 2, "tiny", ["--dropout", "0.1"]),
    # bounded rings: N_m = 12 micro-batches through 8-slot rings, three
    # steps (slots reused within and across steps; AdamW applied between)
    (2, 2, 1, "tiny", ["--N", "12", "--micro-batch", "2", "--steps", "3"]),
    (4, 4, 1, "tiny", ["--N", "10", "--micro-batch", "2", "--steps", "2"]),
    # a user model structure with a CutPoint every 2 layers (modules.GPT2):
    # the stage map covers its CutPoint blocks
    (2, 2, 1, "tiny", ["--cut-every", "2"]),
    # live opportunistic dispatch (StagePolicy on real arrivals)
    (2, 2, 1, "tiny", ["--dispatch", "live", "--steps", "2"]),
    (4, 2, 2, "tiny", ["--dispatch", "live", "--dropout", "0.1"]),
    (4, 4, 1, "tiny", ["--dispatch", "live", "--N", "8", "--micro-batch", "2", "--steps", "2"]),
    (2, 2, 1, "tiny_bert", ["--dropout", "0.1"]),
    # the 8-GPU north-star shapes as 8 ranks on one GPU: 4x2 (355M / 8.3B),
    # 2x4 (BERT-large), 8x1 (2.5B; tiny widened to 8 layers)
    (8, 4, 2, "tiny", []),
    (8, 2, 4, "tiny", []),
    (8, 8, 1, "tiny", ["--layers", "8", "--N", "8", "--micro-batch", "2"]),
    # BASELINE widths, two-layer cuts: 16 MiB (355M, m=1) and 1 MiB-per-row
    # (BERT-large) boundary messages through the rings
    (2, 2, 1, "gpt2_355m", ["--layers", "2", "--micro-batch", "1", "--N", "2"]),
    (4, 2, 2, "bert_large", ["--layers", "2", "--micro-batch", "1", "--N", "2"]),
]


def _ids(c):
    return f"{c[3]}-{c[1]}x{c[2]}-" + "".join(a.strip("-")[:4] for a in c[4])


def _check(p, token):
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    assert token in p.stdout, p.stdout[-4000:]


@pytest.mark.parametrize("case", PIPE_CASES, ids=_ids)
def test_pipeline_matches_oracle_one_gpu(case):
    nproc, P, D, config, extra = case
    _check(launch("dist_pipeline_check.py", nproc,
                  ["--P", P, "--D", D, "--config", config] + extra, same=True), "PARITY OK")


def test_opportunistic_dispatch_one_gpu():
    p = launch("dist_pipeline_check.py", 2, ["--P", 2, "--D", 1, "--dispatch", "opportunistic"],
               same=True)
    _check(p, "PARITY OK")
    moved = [int(x) for x in re.findall(r"differs from static at (\d+) positions", p.stdout)]
    assert len(moved) == 2 and max(moved) > 0, p.stdout[-2000:]


def test_retuned_dispatch_same_losses_one_gpu():
    _check(launch("dist_retune_check.py", 2, same=True), "RETUNE OK")


def test_morph_by_plan_one_gpu():
    _check(launch("dist_morph_check.py", 2, same=True), "MORPH OK")


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.multigpu
@pytest.mark.parametrize("case", [c for c in PIPE_CASES if c[3] in ("tiny", "gpt2_355m",
                                                                     "bert_large")], ids=_ids)
def test_pipeline_matches_oracle_nccl(case):
    nproc, P, D, config, extra = case
    if _gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    _check(launch("dist_pipeline_check.py", nproc,
                  ["--P", P, "--D", D, "--config", config] + extra, same=False), "PARITY OK")


@pytest.mark.multigpu
def test_morph_by_plan_nccl():
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    _check(launch("dist_morph_check.py", 2, same=False), "MORPH OK")
