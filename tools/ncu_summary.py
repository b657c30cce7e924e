"""Summaries of ncu output for profiles/ (no GPU needed).

  python tools/ncu_summary.py launches <launches.csv> <tag>     # per-pass table of one step
  python tools/ncu_summary.py full <report.ncu-rep> <tag>       # key metrics per captured kernel
"""
import csv
import io
import subprocess
import sys

ALG_GB = 8.589934592   # 2 * 4096^2 * 8 B * 32 images per pass (C4)
PASS = {0: "K1", 1: "K2/K4", 2: "K3", 3: "K5", 4: "LC-P1", 5: "LC-P3"}


def launches(path, tag):
    rows = [l for l in open(path) if l.startswith('"')]
    r = list(csv.reader(io.StringIO("".join(rows))))
    h = r[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for row in r[1:]:
        per.setdefault(int(row[ii]), {"k": row[ki]})[row[mi]] = float(row[vi].replace(",", ""))
    ids = sorted(per)
    # the C4 step's kernels (log2 N = 12; the sub-records of other configs launch others)
    ours = [i for i in ids if "nslct" in per[i]["k"] and ("<float, 12," in per[i]["k"] or "<12," in per[i]["k"])]
    last = ours[-5:]   # one step = the last 5 launches
    tot = sum(per[i]["gpu__time_duration.sum"] for i in last)
    print("# %s ncu launch list (bench.py --steps 1 --warmup 3, C4 4096^2 c64 batch 32, 1 B200)" % tag)
    print("# cold-cache, serialised by ncu: compare shares, not absolutes")
    print("pass,kernel,ms,share_of_step,dram_read_GB,dram_write_GB,alg_GB")
    names = ["K1", "K2", "K3", "K4", "K5"]
    for n, i in zip(names, last):
        d = per[i]
        t = d["gpu__time_duration.sum"]
        t_ms = t / 1e6 if t > 1000 else t   # ns or ms depending on ncu units
        rd = d.get("dram__bytes_read.sum", 0)
        wr = d.get("dram__bytes_write.sum", 0)
        print("%s,%s,%.3f,%.3f,%.3f,%.3f,%.3f" % (n, d["k"].split("(")[0], t_ms,
              t / tot, rd / 1e9 if rd > 1e6 else rd, wr / 1e9 if wr > 1e6 else wr, ALG_GB))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic"] + \
       ["smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s for s in
        ("barrier", "mio_throttle", "short_scoreboard", "long_scoreboard", "not_selected", "wait",
         "dispatch_stall", "lg_throttle", "math_pipe_throttle")]


def full(rep, tag):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    print("# %s ncu --set full capture (--clock-control none), one launch per kernel of one step" % tag)
    print("kernel," + ",".join(k.replace("smsp__average_warps_issue_stalled_", "stall_") for k in KEYS))
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0]
        vals = [row[h.index(k)] if k in h else "" for k in KEYS]
        print(name + "," + ",".join(vals))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
