#!/usr/bin/env python
"""Device timeline of one low-rank solve (CUPTI through torch.profiler; the
kernels are this library's, torch only collects the activity records):
per-kernel totals, busy vs idle time of the stream, and the largest gaps.
python tools/lr_timeline.py C2 [C4 ...]   (not a bench: profiler overhead)"""
import collections
import re
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2603_25233_b200 as P  # noqa: E402

def short(n):
    return n.replace("rtlr::cuda::(anonymous namespace)::", "").replace("rtlr::cuda::", "").replace("void ", "")


for name in sys.argv[1:] or ["C2"]:
    sp = P.Problem(name)
    sp.solve_low_rank(build_factors=0)  # warm
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rep = sp.solve_low_rank(build_factors=0)
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", f"lr_timeline_{name}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"]
          if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    os.remove(path)
    ev.sort(key=lambda e: e["ts"])
    t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
    busy, end = 0.0, t0
    gaps = collections.Counter()
    gap_total = collections.defaultdict(float)
    prev = None
    for e in ev:
        s, d = e["ts"], e["dur"]
        if s > end:
            g = s - end
            key = short(prev or "start")[:34] + " -> " + short(e["name"])[:34]
            gaps[key] += 1
            gap_total[key] += g
            busy += d
        else:
            busy += max(0.0, s + d - end)
        end = max(end, s + d)
        prev = e["name"]
    tot = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        k = re.split(r"[<(]", short(e["name"]))[0][-70:]
        tot[k][0] += 1
        tot[k][1] += e["dur"]
    span = (t1 - t0) * 1e-6
    print(f"== {name}: solve {float(rep.get("solve_seconds", 1)[0]):.3f} s (under the profiler), device span {span:.3f} s, "
          f"busy {busy * 1e-6:.3f} s, idle {span - busy * 1e-6:.3f} s, {len(ev)} activities")
    for k, (c, d) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:28]:
        print(f"  {d * 1e-6:8.4f} s {c:7d} x {d / c:9.1f} us  {k}")
    print("  -- idle by transition (top 16)")
    for k, g in sorted(gap_total.items(), key=lambda kv: -kv[1])[:16]:
        print(f"  {g * 1e-6:8.4f} s {gaps[k]:7d} x {g / gaps[k]:9.1f} us  {k}")
