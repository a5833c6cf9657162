#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, on reports brought back
from gpurun_out/).

  python tools/ncu_summary.py full   <report.ncu-rep> <out.txt> [--traffic profiles/traffic.json --kernel lookup]
  python tools/ncu_summary.py launches <launches.csv> <out.txt>

`full`: per profiled kernel: duration, DRAM bytes (read+write = traffic), shared-memory
wavefronts and % of peak, issue-slot utilisation, occupancy, registers, top stall reasons.
`launches`: per-kernel-name launch count, summed and mean gpu__time_duration, and share.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("dram__bytes_read.sum", "dram_read_B"),
    ("dram__bytes_write.sum", "dram_write_B"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefront_pct_peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_cycles_pct"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__cycles_elapsed.avg", "sm_cycles"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fp32_fma_pipe_pct"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy_pipe_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_inst_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_inst_pct"),
]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "second": 1e9}


def raw_rows(rep):
    """Header, units and data rows of the raw page; values converted to bytes / ns."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    data = []
    for r in rows[2:]:
        conv = []
        for v, u in zip(r, units):
            if u in SCALE:
                try:
                    v = repr(float(v.replace(",", "")) * SCALE[u])
                except ValueError:
                    pass
            conv.append(v)
        data.append(conv)
    return hdr, data


def full(rep, out_path, traffic_path=None, kernel=None):
    hdr, rows = raw_rows(rep)
    lines, traffic = [], {}
    for row in rows:
        rec = dict(zip(hdr, row))
        name = rec.get("Kernel Name", "?")
        lines.append(f"== {name}")
        vals = {}
        for key, label in KEYS:
            v = rec.get(key)
            if v not in (None, ""):
                lines.append(f"  {label:28s} {v}")
                try:
                    vals[label] = float(v.replace(",", ""))
                except ValueError:
                    pass
        stalls = []
        for h, v in rec.items():
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v), h.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("  top stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))
        if kernel and (kernel in name or (kernel == "ccm_knn" and "knn" in name)) and "dram_read_B" in vals:
            traffic = {f"{kernel}_dram_bytes_per_launch": vals["dram_read_B"] + vals.get("dram_write_B", 0.0),
                       "source": rep, "kernel": name}
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_path and traffic:
        try:
            with open(traffic_path) as f:
                old = json.load(f)
        except Exception:
            old = {}
        old.update({k: v for k, v in traffic.items() if k.endswith("_per_launch")})
        old.setdefault("sources", {})[kernel] = {"report": traffic["source"], "kernel": traffic["kernel"]}
        old.pop("source", None)
        old.pop("kernel", None)
        with open(traffic_path, "w") as f:
            json.dump(old, f, indent=1)
    print("\n".join(lines))


def launches(csv_path, out_path):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            k = r[ki].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'sum_ms':>10s} {'mean_us':>10s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {t / 1e6:10.3f} {t / n / 1e3:10.1f} {t / tot:7.3f}")
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        tp = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        kn = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tp, kn)
    else:
        launches(sys.argv[2], sys.argv[3])
