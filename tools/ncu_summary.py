"""Summarise an ncu --set full report: per launch the key throughput / occupancy metrics and the
top warp-stall reasons (cycles per issued instruction)."""
import csv
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def main(path):
    if path.endswith(".csv"):  # a raw-page export
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        print("----", d["Kernel Name"][:90])
        for m in METRICS:
            if m in d:
                print(f"   {m:62s} {d[m]:>18s} {u[h.index(m)]}")
        st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(d[k] or 0))
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        st.sort(key=lambda x: -x[1])
        print("   stalls (cycles/issue): " + ", ".join(f"{k}={v:.2f}" for k, v in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
