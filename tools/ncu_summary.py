"""Summarise an ncu --set full report (one kernel) into a small text file for profiles/:
duration, DRAM bytes/throughput, FP64 pipe and issue utilisation, warp-stall shares and the SASS
opcode mix.   python tools/ncu_summary.py <report.ncu-rep> <title> [command]"""
import collections
import csv
import io
import re
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si, ei = h.index("Source"), h.index("Instructions Executed")
    cnt = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ei:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si].strip())
        if m:
            cnt[m.group(2).split(".")[0]] += int(r[ei] or 0)
    return cnt


def main():
    rep, title = sys.argv[1], sys.argv[2]
    cmd = sys.argv[3] if len(sys.argv) > 3 else ""
    v, u = raw(rep)
    f = lambda k: float(v[k].replace(",", ""))
    t_ms = f("gpu__time_duration.sum") * {"ms": 1, "msecond": 1, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}.get(u["gpu__time_duration.sum"], 1)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = f("dram__bytes_read.sum") * scale[u["dram__bytes_read.sum"]]
    wr = f("dram__bytes_write.sum") * scale[u["dram__bytes_write.sum"]]
    print(f"# {title}")
    if cmd:
        print(f"# command: {cmd}")
    print(f"duration_ms                {t_ms:.3f}")
    print(f"dram_read_GB               {rd / 1e9:.3f}")
    print(f"dram_write_GB              {wr / 1e9:.3f}")
    print(f"dram_GBps                  {(rd + wr) / t_ms / 1e6:.1f}")
    for k in ["dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "gpc__cycles_elapsed.avg.per_second"]:
        if k in v:
            print(f"{k:62s} {v[k]} {u.get(k, '')}")
    tot, items = 0.0, []
    for k, x in v.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                items.append((float(x), k[33:]))
                tot += float(x)
            except ValueError:
                pass
    print("## warp stall sampling (share of samples)")
    for x, k in sorted(items, reverse=True)[:10]:
        print(f"stall_{k:30s} {100 * x / tot:5.1f}%")
    cnt = sass(rep)
    n = sum(cnt.values())
    print(f"## SASS opcode mix ({n} warp-instructions)")
    for op, c in cnt.most_common(14):
        print(f"{op:10s} {100 * c / n:5.1f}%")


if __name__ == "__main__":
    main()
