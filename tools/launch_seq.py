"""Per-launch sequence of one step from an ncu launch-list CSV: python tools/launch_seq.py file.csv [step] [regex]"""
import csv
import re
import sys


def short(name):
    name = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    return name.replace(" ", "")


def rows(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((short(d["Kernel Name"]), float(d["Metric Value"]) / 1000.0))
    return out


def step_rows(path, step=10, nsteps=25):
    data = rows(path)
    per = len(data) // nsteps
    return data[step * per:(step + 1) * per]


if __name__ == "__main__":
    seg = step_rows(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 10)
    pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
    for i, (k, t) in enumerate(seg):
        if pat is None or pat.search(k):
            print(f"{i:4d} {t:8.1f}  {k[:90]}")
