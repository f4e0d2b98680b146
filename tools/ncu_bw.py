"""Per-kernel time and DRAM traffic from an ncu launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (CSV): time share, GB/s achieved."""
import collections
import csv
import sys


def main(path, steps):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.defaultdict(dict)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            per[d["ID"]]["name"] = d["Kernel Name"].split("(")[0][:60]
            per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for v in per.values():
        a = agg[v["name"]]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0)
        a[2] += v.get("dram__bytes_read.sum", 0.0)
        a[3] += v.get("dram__bytes_write.sum", 0.0)
    T = sum(a[1] for a in agg.values())
    print(f"launches {len(per)}  total {T / 1e3 / steps:.1f} us/step (ncu-serialised, warm L2)")
    print(f"{'us/step':>9} {'share':>6} {'n/step':>6} {'MB/step':>8} {'GB/s':>7}  kernel")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        mb = (a[2] + a[3]) / 1e6 / steps
        print(f"{a[1] / 1e3 / steps:9.1f} {100 * a[1] / T:5.1f}% {a[0] / steps:6.1f} {mb:8.1f} "
              f"{(a[2] + a[3]) / max(a[1], 1):7.0f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
