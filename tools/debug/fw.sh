python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/configs_bench.py cfg3 cfg2 cfg1 --steps 5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | cut -c1-200
