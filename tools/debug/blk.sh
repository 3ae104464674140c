mkdir -p gpurun_out/blk
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/blk/build.log 2>&1 || { tail -20 gpurun_out/blk/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "block_fused or qcnn16 or plan_specialised or checkpointed" > gpurun_out/blk/pytest.log 2>&1; tail -3 gpurun_out/blk/pytest.log
timeout 300 python tools/pass_times.py cfg3
QF_BLOCK_ADJ=0 timeout 300 python tools/pass_times.py cfg3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/blk/bench.json 2> gpurun_out/blk/bench.err; tail -1 gpurun_out/blk/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3))"
