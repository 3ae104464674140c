#!/bin/bash
# Round-2 evidence: bench line (with CPU baseline), ncu launch list of the bench command,
# ncu --set full of the middle forward / backward pass kernels at the headline batch.
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ps > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/ncu_launch.log
QF_B=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qf_[af]_p2" -c 2 \
  -o $OUT/passes python tools/prof_qaoa.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full.log
cut -c1-300 $OUT/bench.json; tail -1 $OUT/ncu_launch.log; tail -1 $OUT/ncu_full.log
