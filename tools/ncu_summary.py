"""Print the key counters of the first kernel in an ncu report (raw page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
def summarize(h, u, v):

    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    for w in want:
        if w in h:
            i = h.index(w)
            print(f"{w:70s} {u[i]:10s} {v[i]}")
    st = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v[i]), name.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("stalls (warps per issue):", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
    print()


out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
for v in r[2:]:
    summarize(h, u, v)
