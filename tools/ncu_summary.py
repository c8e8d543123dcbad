"""Print the key metrics of an ncu --set full report (one row per profiled kernel)."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    for r in rows[1:]:
        if r[mi] in KEYS:
            print(r[ii], r[ki].split("(")[0][:40], "|", r[mi], r[vi], r[ui])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        for k in RAW:
            if k in h:
                i = h.index(k)
                print(r[h.index("ID")], "|", k, r[i], u[i])
    stalls = [(float(r[i]) if r[i] else 0.0, n) for i, n in enumerate(h) if "average_warps_issue_stalled" in n
              and n.endswith("per_issue_active.ratio") for r in rows[2:3]]
    for v, n in sorted(stalls, reverse=True)[:6]:
        print("stall", n.split("stalled_")[1].split("_per")[0], round(v, 2))


if __name__ == "__main__":
    main(sys.argv[1])
