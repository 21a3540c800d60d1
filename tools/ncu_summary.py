"""Summarise an ncu report (raw page) per kernel launch: time, occupancy,
pipe/smem utilisation, DRAM traffic, top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "inst_tput_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_cmd_read.sum": "smem_read_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
}


def main(path, kfilter=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        if kfilter not in name:
            continue
        print(f"== {name[:90]}")
        vals = []
        for k, short in KEYS.items():
            if k in idx and idx[k] < len(r):
                u = units[idx[k]] if idx[k] < len(units) else ""
                u = "" if u in ("", "%", "register/thread", "inst/cycle") else " " + u
                vals.append(f"{short}={r[idx[k]]}{u}")
        print("   " + "  ".join(vals))
        st = []
        for c in stall_cols:
            try:
                st.append((float(r[idx[c]].replace(",", "")), c.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
        st.sort(reverse=True)
        print("   stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
