"""Per-region stall breakdown of one kernel from an ncu report (source page, SASS).
Usage: python tools/ncu_sass_stalls.py <report.ncu-rep> <kernel regex> [launch index]
Prints the stall reasons summed over the kernel and the top instructions by samples."""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
idx = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0 for c in cols}
per = []
seen = set()
for r in rows[2:]:
    if len(r) < len(h) or not r[h.index("Warp Stall Sampling (All Samples)")].isdigit():
        continue
    d = dict(zip(h, r))
    if d["Address"] in seen:   # the page repeats per source file view
        continue
    seen.add(d["Address"])
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    per.append((s, d["Address"], d["Source"].strip(), {c: int(d[c] or 0) for c in cols}))
    for c in cols:
        tot[c] += int(d[c] or 0)
T = sum(tot.values())
print("# %s: %d samples" % (rows[0][1][:90], T))
for c, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print("%-22s %5.1f%%" % (c, 100.0 * v / T))
print("# top instructions")
for s, a, src, st in sorted(per, key=lambda x: -x[0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    top = sorted(st.items(), key=lambda x: -x[1])[:2]
    print("%5.2f%% %-45s %s" % (100.0 * s / T, src[:45], " ".join("%s=%d" % (k[6:], v) for k, v in top)))
