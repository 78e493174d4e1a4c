"""Measured Alg 1 vs version B crossover against the planner's choice (SURVEY
8(f) rank 3).  For m = 1 .. 64 ciphertexts of 128
Softmax of dim 256 on [-128, 0] (k = 5, P16, the tab:SMmany setting,
PAPER.md 585-600) it runs both variants as CUDA-graph plans on one GPU, times
the replays with CUDA events, and prints one JSON line per (m, variant) with
the measured ms per step, the ledger's bootstrap count and the planner's
prediction (hs_softmax_schedule), then the planner's pick vs the measured
winner.  Usage: python tools/variant_sweep.py [--ms 1,2,4,8,16,64] [--reps 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,2,4,8,16,64")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    tabs = {"A": "p16_n256_M128_k5_A", "B": "p16_n256_M128_k5_B"}
    rows = []
    for m in [int(v) for v in args.ms.split(",")]:
        name = f"sweep_m{m}"
        W.WORKLOADS[name] = dict(preset="P16", n=256, L=128 * m, m=m, M=128.0, k=5, variant="B", table=tabs["B"])
        S = bench.build_setup(name, 0, 1, 0)
        hs, K, B, P, ctx = S["hs"], S["K"], S["B"], S["P"], S["ctx"]
        tables = W.poly_tables()
        cands = [dict(k=5, variant=v, exp=tables[t]["exp"], inv=tables[t]["inv"]) for v, t in tabs.items()]
        best, sched = hs.softmax_choose(P, cands, 256, m, S["in_level"], bts_out_level=S["top"])
        meas = {}
        for (v, t), pl in zip(tabs.items(), sched):
            tab = tables[t]
            plan = hs.Plan(K, S["cts"], 256, m, 5, v, tab["exp"], tab["inv"], bts=B)
            plan.run()
            torch.cuda.synchronize()
            ctx.ledger_reset()
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.reps):
                plan.run()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            led = ctx.ledger()
            meas[v] = ms
            row = {"m": m, "variant": v, "ms_per_step": round(ms, 2), "ms_per_softmax": round(ms / (128 * m), 4),
                   "bts_measured": led["bts"] // args.reps, "bts_planned": pl["bts_main"] + pl["bts_aux"],
                   "planned_cost": round(pl["cost"], 1), "planned_ms": round(pl["cost"] * 0.228, 1)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del plan
        won = min(meas, key=meas.get)
        print(json.dumps({"m": m, "planner_pick": list(tabs)[best], "measured_winner": won,
                          "agree": list(tabs)[best] == won}), flush=True)
        del S, K, B, ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
