"""Per-launch table from an ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv launch list:   python tools/launch_summary.py <launches.csv> <title>"""
import csv
import sys


def main():
    f, title = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "byte": 1, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}
    d = {}
    for r in rows[1:]:
        d.setdefault((int(r[ii]), r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", "")) * scale[r[ui]]
    print(f"# {title} — ncu launch list (serialised, --clock-control none): per-launch time and DRAM traffic")
    tot_t = tot_b = 0.0
    for (i, k), m in sorted(d.items()):
        t = m["gpu__time_duration.sum"]
        b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        tot_t += t
        tot_b += b
        print(f"{i:4d} {k:16s} {t * 1e3:9.3f} ms {b / 1e9:8.2f} GB {b / t / 1e9:8.1f} GB/s")
    print(f"total {tot_t:.4f} s, {tot_b / 1e9:.1f} GB, {tot_b / tot_t / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
