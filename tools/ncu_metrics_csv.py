"""Per-kernel averages from an `ncu --metrics ... --csv --log-file` launch list:
duration, DRAM read+write, L2 (lts) bytes, per distinct (kernel name, grid).

usage: python tools/ncu_metrics_csv.py launches.csv
"""
import collections
import csv
import io
import sys


def main(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    per = collections.OrderedDict()
    for r in rows:
        key = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "") + " " + r["Grid Size"]
        launch = per.setdefault(key, collections.defaultdict(dict))
        launch[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    print(f"{'kernel':50s} {'n':>4s} {'us/launch':>10s} {'DRAM MB':>8s} {'DRAM GB/s':>9s} {'L2 MB':>8s} {'L2 GB/s':>8s}")
    for k, launches in per.items():
        n = len(launches)
        avg = lambda m: sum(v.get(m, 0.0) for v in launches.values()) / n  # noqa: E731
        t = avg("gpu__time_duration.sum") / 1e3
        d = (avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")) / 1e6
        l2 = avg("lts__t_bytes.sum") / 1e6
        print(f"{k:50s} {n:4d} {t:10.1f} {d:8.1f} {d / t * 1e3 if t else 0:9.0f} {l2:8.1f} "
              f"{l2 / t * 1e3 if t else 0:8.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
