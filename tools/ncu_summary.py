"""JSON summary of an ncu --page raw --csv capture: per profiled kernel launch the key
metrics, plus the decode-step totals (sum over the launches of one step) that bench.py
reports as roofline.traffic.

    python tools/ncu_summary.py raw.csv <config> > profiles/<round>/ncu_<config>_summary.json
"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, units = rows[hdr_i], rows[hdr_i + 1]
col = {h: i for i, h in enumerate(hdr)}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "Kbyte/block": 1e3,
         "byte/block": 1}
WANT = {
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "duration_s": "gpu__time_duration.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
}


def num(vals, name):
    v = vals[col[name]].replace(",", "")
    return float(v) * SCALE.get(units[col[name]], 1)


launches = []
for vals in rows[hdr_i + 2:]:
    if len(vals) != len(hdr) or not vals[col["Kernel Name"]]:
        continue
    d = {"kernel": vals[col["Kernel Name"]], "grid": vals[col["Grid Size"]] if "Grid Size" in col else None,
         "block": vals[col["Block Size"]] if "Block Size" in col else None}
    for k, m in WANT.items():
        if m in col:
            try:
                d[k] = num(vals, m)
            except ValueError:
                d[k] = vals[col[m]]
    if "dram_bytes_read" in d and "duration_s" in d:
        d["dram_gbs"] = (d["dram_bytes_read"] + d.get("dram_bytes_write", 0)) / d["duration_s"] / 1e9
    launches.append(d)
tot = {k: sum(x.get(k, 0) for x in launches) for k in ("dram_bytes_read", "dram_bytes_write", "duration_s",
                                                        "inst_executed")}
out = {"config": sys.argv[2], "kernel": " + ".join(x["kernel"] for x in launches), "launches": launches, **tot}
if tot["duration_s"]:
    out["dram_gbs"] = (tot["dram_bytes_read"] + tot["dram_bytes_write"]) / tot["duration_s"] / 1e9
print(json.dumps(out, indent=1))
