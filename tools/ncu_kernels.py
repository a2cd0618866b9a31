"""Per-(kernel, grid) averages of an ncu --metrics ... --csv launch list:
duration, DRAM bytes and GB/s, L2 bytes, DMMA pipe %.

usage: python tools/ncu_kernels.py launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    mi, vi, ki, gi, ii = (H.index(c) for c in ("Metric Name", "Metric Value", "Kernel Name", "Grid Size", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[h + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "")[-34:]
            per[(r[ii], name, r[gi])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(list)
    for (_, k, g), d in per.items():
        agg[(k, g)].append(d)
    print(f"{'kernel':36s} {'grid':>14s} {'n':>3s} {'us':>9s} {'DRAM MB':>9s} {'DRAM GB/s':>9s} {'L2 MB':>9s} {'dmma%':>6s}")
    for (k, g), L in sorted(agg.items()):
        def avg(key):
            return sum(d.get(key, 0.0) for d in L) / len(L)

        t = avg("gpu__time_duration.sum") / 1e3
        dr = (avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")) / 1e6
        dm = avg("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
        print(f"{k:36s} {g:>14s} {len(L):3d} {t:9.1f} {dr:9.1f} {dr / t * 1e3 if t else 0:9.0f} "
              f"{avg('lts__t_bytes.sum') / 1e6:9.1f} {dm:6.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
