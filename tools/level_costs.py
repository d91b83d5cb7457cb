"""Where a V-cycle's time goes, level by level: V-cycles of the sub-hierarchies
levels[k:] (k = 0 .. L-2) of a workload, device-resident, graph replays.  The
difference between consecutive k is what level k adds (its smoothing,
residual, transfers and corrections).

    python tools/level_costs.py [--workload C2]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--reps", type=int, default=300)
    args = ap.parse_args()
    import torch
    from paper_2402_12947_b200 import configs
    from paper_2402_12947_b200.mg import DeviceHierarchy
    h, b_host, _ = configs.build(configs.WORKLOADS[args.workload])
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(len(h.levels) - 1):
        dh = DeviceHierarchy(h.levels[k:], h.coarse_factor)
        n = dh.n[0]
        b = torch.randn(n, dtype=torch.float64, device="cuda")
        u = torch.zeros_like(b)
        for _ in range(10):
            dh.vcycle(b, u)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.reps):
            dh.vcycle(b, u)
        e1.record()
        torch.cuda.synchronize()
        out.append({"from_level": k, "rows": n, "us": round(e0.elapsed_time(e1) / args.reps * 1e3, 2),
                    "launches": dh.launches_per_vcycle()})
    for i in range(len(out)):
        nxt = out[i + 1]["us"] if i + 1 < len(out) else 0.0
        out[i]["level_adds_us"] = round(out[i]["us"] - nxt, 2)
    print(json.dumps({"workload": args.workload, "sub_hierarchies": out}))


if __name__ == "__main__":
    main()
