python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for cfg in "QF_X=0" "QF_GEOM_FWD=11,4" "QF_GEOM_FWD=12,4" "QF_MINB_FWD=3" "QF_MINB_ADJ=1" "QF_GEOM_FWD=12,4 QF_MINB_FWD=2"; do
  echo "$cfg"; env $cfg timeout 300 python tools/pass_times.py cfg3 2>&1 | tail -1 | cut -c1-260
done
