"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count / total / share, and (with --list) every launch in order."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                us = v / 1e3 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1e3
                name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
                name = name.replace("ldgmg_b200::", "").replace("<unnamed>::", "")
                launches.append((name, d.get("Grid Size", ""), us))
    tot = sum(u for _, _, u in launches)
    agg = collections.OrderedDict()
    for n, _, u in launches:
        c, t = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, t + u)
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:48]:48s} n={c:4d} t={t:10.1f}us share={t / tot:.3f}")
    print(f"total {tot:.1f} us over {len(launches)} launches")
    if "--list" in sys.argv:
        for i, (n, gsz, u) in enumerate(launches):
            print(i, n[:40], gsz, f"{u:.1f}")


if __name__ == "__main__":
    main()
