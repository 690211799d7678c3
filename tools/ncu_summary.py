"""Key metrics of an ncu --set full report (raw page) as a small table."""
import csv, subprocess, sys
WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / instr"),
        ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
        ("launch__registers_per_thread", "registers / thread"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block")]
for rep in sys.argv[1:]:
    if rep.endswith(".csv"):  # an exported raw page (ncu -i X --page raw --csv)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    rows = r[2:]
    names = [row[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:40] for row in rows]
    print(f"### {rep}\n")
    print("| metric | " + " | ".join(names) + " |")
    print("|---|" + "---|" * len(rows))
    for k, lab in WANT:
        if k in h:
            i = h.index(k)
            print(f"| {lab} ({u[i]}) | " + " | ".join(row[i] for row in rows) + " |")
    print()
