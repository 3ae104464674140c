#!/bin/bash
# Round-end evidence on one B200: GPU suite, smoke, bench line (CPU baseline + GPU PS leg),
# ncu launch list of the bench command, ncu --set full of the top kernels, tensor-core bench.
OUT=gpurun_out/${1:-final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ps > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/ncu_launch.log
QF_B=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qf_turn|qf_a_p2|qf_f_p2" -c 3 \
  -o $OUT/passes python tools/prof_qaoa.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full.log
timeout 300 python tools/tc_bench.py > $OUT/tc_bench.json 2>&1
cuobjdump -sass paper_2003_02989_b200/libqfb200.so 2>/dev/null | grep -oE "UTCHMMA|LDTM|UTCBAR|SYNCS[A-Z0-9.]*|UTMALDG" | sort | uniq -c > $OUT/tc_sass.txt
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cut -c1-300 $OUT/bench.json; tail -1 $OUT/ncu_launch.log; tail -1 $OUT/ncu_full.log
