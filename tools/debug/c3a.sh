python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for cfg in "QF_GEOM_ADJ=12,3" "QF_GEOM_ADJ=11,4" "QF_MINB_ADJ=3" "QF_GEOM_ADJ=11,3"; do
  echo "$cfg"; env $cfg timeout 300 python tools/pass_times.py cfg3 2>&1 | tail -1 | cut -c1-260
done
