python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out/bd
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/bd/pytest.log 2>&1; tail -1 gpurun_out/bd/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bd/launches.csv python tools/configs_bench.py cfg3 --steps 1 > /dev/null 2>&1; echo ncu=$?
timeout 600 python tools/configs_bench.py cfg3 cfg2 cfg4 --steps 5 | cut -c1-150
