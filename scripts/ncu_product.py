"""Per-product kernel figures from an ncu --set full capture and a launch list.
usage: python scripts/ncu_product.py REP.ncu-rep LAUNCH_SUMMARY.json OUT.json
Groups the captured launches of each kernel (all template instances, e.g. the
gather's first / accumulate / final windows) and scales their mean by the
kernel's launches per product (the launch list of one step)."""
import json
import subprocess
import sys

rep, ls_path, out_path = sys.argv[1:4]
summ = json.loads(subprocess.run([sys.executable, "scripts/ncu_summary.py", rep],
                                 capture_output=True, text=True, check=True).stdout)
steps = {k.split("::")[-1]: v for k, v in json.load(open(ls_path))["step_launch_counts"].items()}
groups = {}
for name, ents in summ.items():
    groups.setdefault(name.split("<")[0].split("::")[-1], []).extend(ents)
res = {"source": f"{rep} (ncu --set full --clock-control none); launches per product from "
                 f"{ls_path}", "kernels": {}}
for short, ents in groups.items():
    mean = {k: sum(e.get(k, 0.0) for e in ents) / len(ents)
            for k in ents[0] if k != "top_stalls"}
    lp = steps.get(short, 0)
    dram = mean.get("dram_read", 0.0) + mean.get("dram_write", 0.0)
    res["kernels"][short] = {
        "captured_launches": len(ents), "launches_per_product": lp,
        "time_ms_per_launch": mean.get("time_ms"),
        "dram_bytes_per_launch": dram, "dram_bytes_per_product": dram * lp,
        "tensor_pipe_pct": mean.get("tensor_pipe_pct"), "fp64_pipe_pct": mean.get("fp64_pipe_pct"),
        "issue_pct": mean.get("issue_pct"), "dram_pct": mean.get("dram_pct"),
        "l1tex_pct": mean.get("l1tex_pct"), "regs": mean.get("regs"),
        "smem_conflicts_per_launch": mean.get("smem_conflicts"),
        "top_stalls": ents[0]["top_stalls"]}
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
