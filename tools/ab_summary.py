"""Summarise an A/B job directory: trace_*.jsonl (tools/trace_phases.py) and ab_solve.log (tools/ab_solve.py)."""
import collections
import glob
import json
import os
import sys

d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "trace_*.jsonl"))):
    print("==", os.path.basename(f))
    for line in open(f):
        j = json.loads(line)
        k = j["kernels"]
        b = [x for x in k if x.startswith("k_bwd")][0]
        print(" ", j["shape"], b, "span", k[b]["span_us"], "phases", k[b]["phase_mean_us"], "max", k[b]["phase_max_us"],
              "| fwd span", k["k_fwd"]["span_us"], "| gram tail", k.get("gram_tail_last_cta", {}).get("phases_us_median"),
              "| gaps", j["gaps_us_median"], "| us/iter", round(j["solve_span_us"] / j["iters"], 1))
p = os.path.join(d, "ab_solve.log")
if os.path.exists(p):
    r = collections.defaultdict(list)
    for line in open(p):
        if line.startswith("{"):
            j = json.loads(line)
            r[(j["shape"], j["lib"])].append((round(j["iters_per_s_median"], 1), j["runs"][0]["iters"], j["runs"][0]["x_sum"]))
    for k in sorted(r):
        print(k, r[k])
