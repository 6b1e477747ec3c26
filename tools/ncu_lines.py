"""Warp-stall samples per CUDA source line of one kernel in an ncu --set full report
(`--page source --print-source cuda,sass`), largest first:  python tools/ncu_lines.py REP [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, fname, hdr, cur = {}, "", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0] not in ("", "-"):            # a CUDA line row starts a group
        cur = (fname, r[0], r[1][:90])
    if r[2] not in ("", "-") and cur is not None:   # a SASS row under the current line
        try:
            smp = int(r[4])
        except ValueError:
            continue
        agg[cur] = agg.get(cur, 0) + smp
tot = sum(agg.values()) or 1
print(f"total warp-stall samples: {tot}")
for (f, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100.0 * v / tot:6.2f}%  {f}:{ln}  {src}")
