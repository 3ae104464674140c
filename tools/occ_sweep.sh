mkdir -p gpurun_out/occ
for v in "" "QF_SMEM_PAD_FWD=60000" "QF_SMEM_PAD_FWD=80000" "QF_SMEM_PAD_FWD=110000"; do
  env $v timeout 600 python tools/configs_bench.py cfg4 --steps 3 --no-cpu > "gpurun_out/occ/cfg4_$(echo ${v:-base} | tr '=' '_').json" 2>&1
done
AB_TAG=occ3 AB_CFG=cfg3 bash tools/ab.sh "QF_LANE_OPS=0"
for f in gpurun_out/occ/*.json; do echo "$f $(tail -1 $f | cut -c1-120)"; done
