python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out/c3b
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/c3b/pytest.log 2>&1; tail -2 gpurun_out/c3b/pytest.log
timeout 600 python tools/configs_bench.py cfg3 cfg2 --steps 5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3b/launches.csv python tools/configs_bench.py cfg3 --steps 1 > /dev/null 2>&1; echo ncu=$?
