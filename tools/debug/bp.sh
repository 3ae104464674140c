python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "block or qcnn or plan_specialised" 2>&1 | tail -2
timeout 300 python tools/pass_times.py cfg3 | cut -c1-220
