bash tools/gpu_quick.sh ck1
QF_CKPT=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ck1/bench0.json 2>&1; tail -1 gpurun_out/ck1/bench0.json | cut -c1-300
