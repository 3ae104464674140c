python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for cfg in "QF_X=0" "QF_MINB_FWD=3" "QF_MINB_FWD=5" "QF_MINB_FWD=6" "QF_GEOM_FWD=12,4"; do
  echo "$cfg $(env $cfg timeout 300 python tools/configs_bench.py cfg4 --steps 3 2>&1 | tail -1 | cut -c40-120)"
done
