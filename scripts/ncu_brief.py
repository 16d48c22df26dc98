"""Brief of one ncu --set full report (first kernel): duration, DRAM, issue, stalls."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:90])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "smsp__warps_active.avg.per_cycle_active", "launch__grid_size"]:
        print(f"  {k:60s} {d.get(k)}")
    st = {k.split("stalled_")[1].split("_per")[0]: float(d[k]) for k in d
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio") and d[k]}
    print("  stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0.05))
