#!/bin/bash
# ncu --set full of selected tile-pass kernels (QAOA 20q, B=32) under given env.
# usage: tools/ncu_passes.sh TAG KERNEL_REGEX [VAR=VAL ...]
TAG=$1; KRE=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
env "$@" QF_B=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 4 \
  -o $OUT/passes python tools/prof_qaoa.py > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_full.log
tail -2 $OUT/ncu_full.log
