"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel share of device time
    python tools/ncu_summary.py details <report.ncu-rep>     # key --set full metrics per kernel
    python tools/ncu_summary.py kernels <rep.ncu-rep>...     # duration, DRAM GB/s vs the HBM peak, SM%
"""

import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'kernel':64s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:64]:64s} {v[0]:8d} {v[1] / 1e6:10.3f} {v[1] / 1e3 / v[0]:10.1f} {100 * v[1] / tot:6.2f}%")


KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            print(f"{d['Kernel Name'].split('(')[0][:50]:50s} {d['Metric Name']:36s} "
                  f"{d['Metric Value']:>14s} {d['Metric Unit']}")
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) > 2:
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            for k in RAW:
                if k in d:
                    print(f"{d.get('Kernel Name', '?').split('(')[0][:50]:50s} {k:60s} {d[k]:>16s} {u[k]}")


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
          "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
          "ms": 1e-3, "s": 1.0,
          "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
          "cycle/second": 1.0}


def kernels(*reps, hbm_peak=6542.4):
    """Per kernel (longest launch in each capture): duration, DRAM bytes and
    GB/s against the measured HBM peak, SM and memory throughput (% of peak)."""
    print(f"{'kernel':34s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>8s} {'%HBM':>6s} {'SM%':>6s} {'Mem%':>6s} {'GHz':>5s}")
    for rep in reps:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]

        def val(r, k):
            if k not in hdr:
                return 0.0
            i = hdr.index(k)
            try:
                return float(r[i].replace(",", "")) * _SCALE.get(units[i], 1.0)
            except ValueError:
                return 0.0

        best = collections.OrderedDict()
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
            t = val(r, "gpu__time_duration.sum")
            if name not in best or t > best[name][0]:
                best[name] = (t, val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                              val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                              val(r, "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
                              val(r, "sm__cycles_elapsed.avg.per_second"))
        for name, (t, b, sm, mem, hz) in best.items():
            gbs = b / t / 1e9 if t else 0.0
            print(f"{name[:34]:34s} {t * 1e6:9.1f} {b / 1e6:9.1f} {gbs:8.1f} {100 * gbs / hbm_peak:6.1f} "
                  f"{sm:6.1f} {mem:6.1f} {hz / 1e9:5.2f}")


if __name__ == "__main__":
    {"launches": launches, "details": details, "kernels": kernels}[sys.argv[1]](*sys.argv[2:])
