"""Top stalled SASS instructions of one kernel in an ncu report."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "-s", "0", "-c", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
recs = []
tot = 0
for r in rows[1:]:
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"])
    except Exception:
        continue
    tot += s
    recs.append((s, d["Address"][-5:], d["Source"].strip()))
for s, a, src in sorted(recs, reverse=True)[:top]:
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}%  {a}  {src}")
print("total samples", tot)
