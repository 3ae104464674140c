#!/bin/bash
# Full GPU check: parity suite, smoke, bench, per-config timings.
OUT=gpurun_out/${1:-full}
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python tools/configs_bench.py --steps 3 > $OUT/configs.jsonl 2>&1
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cut -c1-400 $OUT/bench.json; cut -c1-250 $OUT/configs.jsonl
