"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections
import csv
import sys


def summarize(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        name = d["Kernel Name"].split("(")[0][:70]
        tot[name] += float(d["Metric Value"])
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"launches: {len(data)}  total: {T/1000:.1f} us (ncu-serialised, cold cache)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"{v/1000:9.1f} us {100*v/T:5.1f}%  n={cnt[k]:3d}  avg {v/cnt[k]/1000:7.1f} us  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
