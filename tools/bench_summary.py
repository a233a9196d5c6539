#!/usr/bin/env python
"""Prints the headline and the solver / phase table of a bench.py JSON line:
python tools/bench_summary.py gpurun_out/bench.log"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(f"{d['value'] / 1e9:.1f} G upd/s, {d['ms_per_step']:.2f} ms/step, frac {r['frac']:.3f} (isolated {r['frac_isolated']:.3f}), "
      f"e2e {d['e2e']['value'] / 1e9:.2f} G upd/s, cpu 1 core {d['cpu_baseline']['value'] / 1e6:.1f} M, clocks {d['clocks']}")
for k, v in d.get("solvers", {}).items():
    if not isinstance(v, dict):
        continue
    print(k, v.get("time_to_tol_s"), v.get("time_to_tol_runs_s"), "rank", v.get("final_rank"), "it", v.get("iterations"),
          ("cpu " + json.dumps(v["cpu_reference"])) if "cpu_reference" in v else "")
    for ph, w in v.get("phases", {}).items():
        if isinstance(w, dict) and "seconds" in w:
            print(f"    {ph:12s} {w['seconds']:.3f} s  calls {w.get('calls')}  hbm {w.get('frac_hbm', 0):.2f}  dmma {w.get('frac_fp64_tensor', 0):.2f}")
