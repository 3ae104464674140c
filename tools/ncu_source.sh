#!/bin/bash
# ncu --set full with per-line source attribution of the generated pass kernels:
# the NVRTC sources are dumped into the working directory so --import-source finds them.
# usage: tools/ncu_source.sh TAG KERNEL_REGEX
TAG=$1; KRE=$2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
rm -rf /root/.cache/qfb200
QF_JIT_DUMP=. QF_B=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 2 \
  -o $OUT/src python tools/prof_qaoa.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu.log
ncu -i $OUT/src.ncu-rep --page source --csv --print-source cuda > $OUT/source.csv 2>/dev/null
tail -2 $OUT/ncu.log
