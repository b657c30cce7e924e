"""SASS opcode mix of one kernel from an ncu report (source page): executed warp
instructions per opcode, normalised per thread-group of a pipe pass.
Usage: python tools/ncu_opmix.py <report.ncu-rep> <kernel regex> [groups per launch]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
groups = int(sys.argv[3]) if len(sys.argv) > 3 else 32 * 4096 // 2   # C4: batch 32, 2-line groups
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
seen, cnt, tot = set(), collections.Counter(), 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    d = dict(zip(h, r))
    if d["Address"] in seen or not d["Instructions Executed"].isdigit():
        continue
    seen.add(d["Address"])
    n = int(d["Instructions Executed"])
    tot += n
    op = d["Source"].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    cnt[op.split()[0].split(".")[0]] += n
print("# %s: %d warp instructions; per thread-group (16 compute warps) below" % (rows[0][1][:80], tot))
for k, v in cnt.most_common(40):
    print("%-12s %8.1f  %5.1f%%" % (k, v / groups / 16, 100.0 * v / tot))
