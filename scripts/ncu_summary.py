"""Summarise an ncu report: per kernel time, DRAM bytes, pipes, stalls."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "smem_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
scale = {"ms": 1.0, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "msecond": 1.0,
         "second": 1e3}
byte_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    short = short.replace("nld::mma::", "").replace("nld::", "").replace("unnamed>::", "")
    ent = {}
    for k, h in keys.items():
        if h not in hdr:
            continue
        i = hdr.index(h)
        try:
            v = float(r[i])
        except ValueError:
            continue
        u = units[i]
        if k == "time_ms":
            v *= scale.get(u, 1.0)
        if k.startswith("dram_") and u in byte_scale:
            v *= byte_scale[u]
        ent[k] = v
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                stalls[h.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = float(r[i])
            except ValueError:
                pass
    ent["top_stalls"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:5])
    out.setdefault(short, []).append(ent)
print(json.dumps(out, indent=1))
