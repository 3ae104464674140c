#!/bin/bash
# One GPU-box session: parity suite, bench line, ncu launch list, ncu --set full of the top kernels.
# usage: tools/gpu_round.sh TAG [skip-tests]
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/ncu_launch.log
QF_B=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qf_[af]_p -c 12 \
  -o $OUT/passes python tools/prof_qaoa.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full.log
timeout 900 python tools/configs_bench.py --steps 3 > $OUT/configs.jsonl 2>&1
timeout 600 ncu --set full --clock-control none -k regex:qf_f_p -c 3 -o $OUT/rcs python tools/configs_bench.py cfg4 --steps 1 > $OUT/ncu_rcs.log 2>&1
ls -la $OUT
