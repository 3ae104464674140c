mkdir -p gpurun_out/blk2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/blk2/build.log 2>&1 || { tail -20 gpurun_out/blk2/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/blk2/pytest.log 2>&1; tail -3 gpurun_out/blk2/pytest.log
timeout 300 python tools/pass_times.py cfg3
timeout 300 python tools/pass_times.py cfg1
QF_BLOCK_ADJ=0 timeout 300 python tools/pass_times.py cfg1
timeout 600 python tools/configs_bench.py cfg3 cfg1 --steps 5
