#!/bin/bash
# End-of-round verification on one B200 (builder-side): smoke, the GPU test
# suite, the default bench line and the reference arm, the bench's ncu launch
# list. Output under gpurun_out/$TAG_*.
TAG=${1:-verify}
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.txt 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --launch-skip 6000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --side-dropout 0 \
  --cpu-sample-s 1 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
