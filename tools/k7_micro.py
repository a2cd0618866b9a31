"""K7 (fused ALM update, alm_tma_k) microbenchmark at the RPCA configs.

Event-timed average of one launch on seeded inputs, against the roofline
max(2 m^2 r / DMMA peak, 32 m^2 / HBM peak) (D, Y read; Y', W written). The
E-only end-of-solve pass is timed too (24 B / element: D, Y read, E written).

usage: python tools/k7_micro.py [C3] [C5] [C1] ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402

CFG = {"C1": (500, 25), "C3": (2000, 100), "C3r110": (2000, 110), "C5": (40000, 400), "C5r100": (40000, 100)}


def peaks(ctx):
    dmma = ctx.fp64_peak(0)
    hbm = None
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        for k, v in j.items():
            if "hbm" in k.lower() and isinstance(v, (int, float)):
                hbm = float(v)
                break
    return dmma, hbm or 6553.6


def main():
    ctx = B.Context(0)
    dmma, hbm = peaks(ctx)
    names = sys.argv[1:] or ["C3", "C5"]
    for name in names:
        m, r = CFG[name]
        reps = 3 if m > 10000 else 20
        d = ctx.microbench(11, m, r, reps, detail=True)
        de = ctx.microbench(12, m, r, reps, detail=True)
        us = d[0]
        flop = 2.0 * m * m * r
        byt = 32.0 * m * m
        t_t = flop / (dmma * 1e12) * 1e6
        t_b = byt / (hbm * 1e9) * 1e6
        roof = max(t_t, t_b)
        print(json.dumps({"config": name, "m": m, "r": r, "k7_us": round(us, 2), "roofline_us": round(roof, 2),
                          "bound": "tensor" if t_t >= t_b else "hbm", "frac": round(roof / us, 3),
                          "tflops": round(flop / us / 1e6, 2), "GBps": round(byt / us / 1e3, 1),
                          "eonly_us": round(de[0], 2), "checksum": d[1], "dmma_peak": round(dmma, 2),
                          "hbm_peak": hbm}), flush=True)


if __name__ == "__main__":
    main()
