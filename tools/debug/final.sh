mkdir -p gpurun_out/fin
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fin/pytest.log 2>&1; tail -2 gpurun_out/fin/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; tail -1 gpurun_out/fin/bench.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 2>/dev/null | tail -1 | cut -c1-200
timeout 900 python tools/configs_bench.py --steps 3 | cut -c1-170
