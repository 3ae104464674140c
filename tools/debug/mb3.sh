python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/pass_times.py cfg3 | cut -c1-200
timeout 900 python tools/configs_bench.py cfg3 cfg2 cfg4 cfg5 --steps 3 | cut -c1-160
