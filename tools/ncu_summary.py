"""Per-kernel summary of an ncu --set full report (read with ncu -i --page raw).

usage: python tools/ncu_summary.py report.ncu-rep
Prints, per launch: duration, DRAM bytes read+write, DRAM / SM / tensor
throughput %, registers, achieved occupancy, and the sum over launches.
"""
import csv
import io
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "launch__grid_size": "grid",
}
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"name": r[h.index("Kernel Name")].split("(")[0][-60:]}
        for m, key in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    d[key] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    d[key] = None
        if d.get("dur_us") is not None and units[h.index("gpu__time_duration.sum")] == "ns":
            pass
        res.append(d)
    return res


def main(path):
    rows = load(path)
    tot_t = tot_b = 0.0
    print(f"{'kernel':60s} {'us':>8s} {'DRAM MB':>8s} {'GB/s':>7s} {'mem%':>5s} {'sm%':>5s} {'fp64%':>5s} {'dmma%':>5s} {'regs':>4s} {'occ%':>5s} grid")
    for d in rows:
        b = (d.get("dram_rd") or 0) + (d.get("dram_wr") or 0)
        t = d.get("dur_us") or 0
        tot_t += t
        tot_b += b
        print(f"{d['name']:60s} {t:8.1f} {b / 1e6:8.2f} {b / max(t, 1e-9) / 1e3:7.0f} {d.get('mem_pct') or 0:5.1f} "
              f"{d.get('sm_pct') or 0:5.1f} {d.get('fp64_pipe_pct') or 0:5.1f} {d.get('dmma_pct') or 0:5.1f} "
              f"{int(d.get('regs') or 0):4d} "
              f"{d.get('occ_pct') or 0:5.1f} {int(d.get('grid') or 0)}")
    print(f"TOTAL {len(rows)} launches: {tot_t:.1f} us, DRAM {tot_b / 1e6:.2f} MB ({tot_b:.0f} bytes)")


if __name__ == "__main__":
    main(sys.argv[1])
