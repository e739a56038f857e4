"""Summarise an ncu --csv launch list (gpu__time_duration.sum + optional metrics): per kernel
launch in order, or per kernel family totals with --families.
    python tools/launch_table.py gpurun_out/x/launches.csv [--families] [--last N]"""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    k = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = k.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(k.values())


def main():
    launches = load(sys.argv[1])
    if "--last" in sys.argv:
        launches = launches[-int(sys.argv[sys.argv.index("--last") + 1]):]
    if "--families" in sys.argv:
        fam = OrderedDict()
        for l in launches:
            n = l["name"].split("(")[0].split("::")[-1].split("<")[0]
            f = fam.setdefault(n, [0.0, 0])
            f[0] += l["gpu__time_duration.sum"] / 1e3
            f[1] += 1
        for n, (us, c) in fam.items():
            print(f"{n:40s} {c:5d} launches {us:12.1f} us")
        return
    for l in launches:
        extra = " ".join(f"{k.split('.')[0].split('__')[-1]}={v:.4g}" for k, v in l.items()
                         if k not in ("name", "gpu__time_duration.sum"))
        print(f"{l['gpu__time_duration.sum'] / 1e3:10.1f} us  {l['name'][:60]:60s} {extra}")


if __name__ == "__main__":
    main()
