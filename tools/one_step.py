"""One config-3 step for profilers (dev tool, GPU): builds the bench setup and
the CUDA-graph plan (eager warm-up + capture happen OUTSIDE the profiled
range), then replays the plan once between cudaProfilerStart/Stop, so
`ncu --profile-from-start off ...` sees exactly one step's kernels.

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python tools/one_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench


def main():
    torch.cuda.set_device(0)
    S = bench.build_setup("config3", 0, 1, 0)
    hs, K, B, tab, wl = S["hs"], S["K"], S["B"], S["tab"], S["wl"]
    plan = hs.Plan(K, S["cts"], S["n"], S["m"], S["k"], wl["variant"], tab["exp"], tab["inv"], bts=B)
    plan.run()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    plan.run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("one step replayed", file=sys.stderr)


if __name__ == "__main__":
    main()
