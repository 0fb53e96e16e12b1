"""Key metrics + stall mix of every kernel in an ncu report (ncu -i ... --page raw --csv)."""
import csv, io, subprocess, sys
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    print("==", vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w} = {vals[i]} {units[i]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(vals[i].replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in st) or 1
    st.sort(key=lambda x: -x[1])
    print("  stall mix: " + ", ".join(f"{h} {100*v/tot:.1f}%" for h, v in st[:8]))
