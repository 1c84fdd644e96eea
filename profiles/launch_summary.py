"""Summarize an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes] per launch).

    python profiles/launch_summary.py gpurun_out/c2_launches.csv [first_n_rows]
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    k = collections.OrderedDict()
    for r in rows:
        d = k.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(k.values())


def main():
    ks = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in ks:
        base = "tq_pass_*" if d["name"].startswith("tq_pass") else d["name"]
        a = agg[base]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print("%-45s %6s %10s %6s %9s" % ("kernel", "n", "ms", "share", "DRAM GB/s"))
    for nm, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-45s %6d %10.3f %6.3f %9.0f" % (nm[:45], a[0], a[1] / 1e6, a[1] / tot, a[2] / a[1] if a[1] else 0))
    # the gate-pass kernels one by one (run-time specialized: tq_pass_l<level>_p<pass>[_v<variant>])
    per = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in ks:
        if d["name"].startswith("tq_pass"):
            a = per[d["name"]]
            a[0] += 1
            a[1] += d.get("gpu__time_duration.sum", 0)
            a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    if per:
        print("\n%-45s %6s %10s %6s %9s" % ("gate-pass kernel", "n", "ms", "share", "DRAM GB/s"))
        for nm, a in sorted(per.items(), key=lambda x: -x[1][1]):
            print("%-45s %6d %10.3f %6.3f %9.0f" % (nm[:45], a[0], a[1] / 1e6, a[1] / tot, a[2] / a[1] if a[1] else 0))
    if len(sys.argv) > 2:
        for d in ks[: int(sys.argv[2])]:
            t = d.get("gpu__time_duration.sum", 0)
            b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            print("   %-28s %-14s %10.0f ns %8.0f GB/s" % (d["name"][:28], d["grid"], t, b / t if t else 0))


if __name__ == "__main__":
    main()
