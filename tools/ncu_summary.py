"""JSON summary of one ncu --page raw --csv capture (first kernel): the numbers bench.py
reports as roofline.traffic and the judge-facing key metrics.

    python tools/ncu_summary.py raw.csv <config> > profiles/<round>/ncu_<config>_summary.json
"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, units, vals = rows[hdr_i], rows[hdr_i + 1], rows[hdr_i + 2]
col = {h: i for i, h in enumerate(hdr)}


def num(name):
    v = vals[col[name]].replace(",", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
             "Kbyte/block": 1e3, "byte/block": 1}.get(units[col[name]], 1)
    return float(v) * scale


want = {
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "duration_s": "gpu__time_duration.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
}
out = {"config": sys.argv[2], "kernel": vals[col["Kernel Name"]], "grid": vals[col.get("Grid Size", 0)],
       "block": vals[col.get("Block Size", 0)]}
for k, m in want.items():
    if m in col:
        try:
            out[k] = num(m)
        except ValueError:
            out[k] = vals[col[m]]
if "dram_bytes_read" in out and "duration_s" in out:
    out["dram_gbs"] = (out["dram_bytes_read"] + out.get("dram_bytes_write", 0)) / out["duration_s"] / 1e9
print(json.dumps(out, indent=1))
