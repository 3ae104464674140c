python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "parameter_shift or ps or layer or evaluator or stochastic or sampled or install or golden" 2>&1 | tail -3
timeout 600 python tools/configs_bench.py cfg1 --steps 5
python tools/debug/ps_prof.py 2>&1 | head -22
