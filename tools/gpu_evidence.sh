#!/bin/bash
# Round evidence on one B200: GPU suite, smoke, bench line, ncu launch list of the bench command,
# ncu --set full of the headline's pass kernels (+ SASS source page of the backward middle pass),
# every config next to its CPU reference, tensor-core bench, crossbar microbenchmark.
OUT=gpurun_out/${1:-ev}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ps > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/ncu_launch.log
QF_B=256 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"qf_turn|qf_a_p2|qf_a_p4|qf_f_p0|qf_f_p2" -c 5 \
  -o $OUT/passes python tools/prof_qaoa.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full.log
python tools/ncu_summary.py $OUT/passes.ncu-rep > $OUT/ncu_full_passes.txt 2>&1
ncu -i $OUT/passes.ncu-rep --page source --csv --kernel-name regex:qf_a_p2 --print-source sass > $OUT/a_p2_src.csv 2>/dev/null
python tools/ncu_regions.py $OUT/a_p2_src.csv > $OUT/a_p2_regions.txt 2>&1
timeout 2400 python tools/configs_bench.py --steps 3 > $OUT/configs.jsonl 2> $OUT/configs.err
timeout 300 python tools/tc_bench.py > $OUT/tc_bench.json 2>&1
tools/micro/xbar_bench > $OUT/xbar.json 2>&1
tools/micro/ffma2_bench > $OUT/ffma2_bench.json 2>&1
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cut -c1-300 $OUT/bench.json; tail -1 $OUT/ncu_launch.log; tail -1 $OUT/ncu_full.log
