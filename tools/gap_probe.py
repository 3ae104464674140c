"""Device time of one execute() vs the sum of its kernels (torch.profiler / CUPTI), to find
idle gaps between launches.  python tools/gap_probe.py cfg3|cfg2"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from pass_times import bound_for  # noqa: E402


def step_fn(cfg):
    if cfg == "cfg1ps":   # parameter shift: 1024 x 241 shifted circuits through the public API
        from paper_2003_02989_b200 import ops
        from paper_2003_02989_b200 import workloads as wl
        from paper_2003_02989_b200.circuit import circuit_symbols

        circ = wl.hea_circuit(10, 4)
        syms = circuit_symbols(circ)
        th = torch.as_tensor(wl.hea_params(1024)).cuda()
        obs = [wl.z_sum(10)]
        return lambda: ops.expectation_and_ps_gradient(circ, syms, th, obs)
    b, th = bound_for(cfg)
    return lambda: b.execute(th, want_grad=True)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    fn = step_fn(cfg)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print("event ms/step", e0.elapsed_time(e1) / 5)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    tot = sum(e.device_time_range.elapsed_us() if hasattr(e, "device_time_range") else e.cuda_time for e in evs)
    print("kernel sum ms/step", tot / 3 / 1000)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))


if __name__ == "__main__":
    main()
