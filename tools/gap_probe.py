"""Device time of one execute() vs the sum of its kernels (torch.profiler / CUPTI), to find
idle gaps between launches.  python tools/gap_probe.py cfg3|cfg2"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from pass_times import bound_for  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    b, th = bound_for(cfg)
    for _ in range(3):
        b.execute(th, want_grad=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        b.execute(th, want_grad=True)
    e1.record()
    torch.cuda.synchronize()
    print("event ms/step", e0.elapsed_time(e1) / 5)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            b.execute(th, want_grad=True)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    tot = sum(e.device_time_range.elapsed_us() if hasattr(e, "device_time_range") else e.cuda_time for e in evs)
    print("kernel sum ms/step", tot / 3 / 1000)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))


if __name__ == "__main__":
    main()
