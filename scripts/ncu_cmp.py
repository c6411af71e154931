"""Side-by-side key metrics of the kernels in several ncu reports: python scripts/ncu_cmp.py A.ncu-rep B.ncu-rep"""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print("==", rep)
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        vals = [r[h.index(k)] if k in h else "-" for k in KEYS]
        print(name[:48], " ".join(vals))
print("cols:", " | ".join(k.split(".")[0].replace("l1tex__", "") for k in KEYS))
