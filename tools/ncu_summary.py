"""Summarise one ncu --set full report (first kernel) into a text file for profiles/:
key raw metrics and the SOL / memory / scheduler / occupancy sections."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Scheduler Statistics", "Occupancy",
            "Warp State Statistics", "Compute Workload Analysis")


def main(rep, title, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    lines = [f"# ncu --set full capture: {title}", ""]
    lines += [f"{k} = {v[h.index(k)]} {u[h.index(k)]}" for k in KEYS if k in h]
    lines.append("")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(det)))
    for row in rows:
        if row["ID"] == rows[0]["ID"] and row["Section Name"] in SECTIONS:
            lines.append(f"{row['Section Name']} | {row['Metric Name']} = {row['Metric Value']} {row['Metric Unit']}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
