"""Condense `ncu --page raw --csv` exports into the committed evidence:

    python tools/ncu_summarize.py <name> <raw.csv> [alg_bytes] [launch description]

writes profiles/<name>.csv (the metrics below, one per line) and updates the
<kernel> entry of profiles/ncu_summary.json (DRAM traffic vs algorithmic bytes,
shared-memory wavefronts / bank conflicts, tensor pipe, issue, stall samples).
"""

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = (
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
)
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    name, path = sys.argv[1], sys.argv[2]
    alg = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] else None
    desc = sys.argv[4] if len(sys.argv) > 4 else ""
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, vals = rows[start], rows[start + 1], rows[start + 2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    out = os.path.join(ROOT, "profiles", f"{name}.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "value", "unit"])
        for k in KEEP + tuple(sorted(k for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                                     and not k.endswith("_not_issued"))):
            if k in d:
                w.writerow([k, d[k][0], d[k][1]])

    def num(k):
        v, u = d.get(k, ("0", ""))
        try:
            return float(v.replace(",", "")) * SCALE.get(u, 1)
        except ValueError:
            return None

    kern = d["Kernel Name"][0].replace("void ", "").split("<")[0].split("(")[0].replace("vqb::", "").replace("_kernel", "")
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    dram = (num("dram__bytes_read.sum") or 0) + (num("dram__bytes_write.sum") or 0)
    summ[kern] = {
        "capture": f"profiles/{name}.csv", "launch": desc, "alg_bytes": alg, "dram_bytes": int(dram),
        "dram_over_alg": round(dram / alg, 4) if alg else None,
        "duration_us_cold": num("gpu__time_duration.sum"),
        "sm_active_over_elapsed": round(num("sm__cycles_active.avg") / num("gpc__cycles_elapsed.max"), 3),
        "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_wavefront_pct_of_peak": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "smem_ld_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        "smem_st_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
        "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
    }
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(kern, json.dumps(summ[kern]))


if __name__ == "__main__":
    main()
