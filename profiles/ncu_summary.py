"""Summarise an ncu report (raw page) into the metrics we track; optional
--source prints the top stall sites.  Usage: python profiles/ncu_summary.py rep [--source]"""
import csv
import io
import re
import subprocess
import sys

KEYS = [r"gpu__time_duration.sum", r"dram__bytes_read.sum$", r"dram__bytes_write.sum$",
        r"sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        r"sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        r"sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        r"smsp__issue_active.avg.pct_of_peak_sustained_active", r"sm__throughput.avg.pct_of_peak_sustained_elapsed",
        r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$", r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$",
        r"l1tex__data_pipe_lsu_wavefronts_mem_shared_op_(ld|st).sum$", r"lts__throughput.avg.pct_of_peak_sustained_elapsed",
        r"lts__t_bytes.sum$", r"dram__throughput.avg.pct_of_peak_sustained_elapsed",
        r"l1tex__throughput.avg.pct_of_peak_sustained_active", r"launch__registers_per_thread$",
        r"smsp__average_warps_issue_stalled_(long_scoreboard|barrier|wait|short_scoreboard|mio_throttle|lg_throttle|math_pipe_throttle|branch_resolving)_per_issue_active.ratio",
        r"sm__cycles_elapsed.avg$", r"smsp__inst_executed.sum$", r"l1tex__data_pipe_tc_wavefronts_mem_shared.*sum$",
        r"sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", r"launch__grid_size", r"launch__block_size"]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
        print("==", d.get("Kernel Name", "")[:90])
        for k in hdr:
            if any(re.search(p, k) for p in KEYS):
                print(f"  {k} = {d[k]} {u[k]}")
    if "--source" in sys.argv:
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        r = list(csv.reader(io.StringIO(src)))
        h = r[1]; data = r[2:]
        i_s = h.index("Warp Stall Sampling (All Samples)"); i_src = h.index("Source")
        tot = sum(float(x[i_s] or 0) for x in data) or 1
        for x in sorted(data, key=lambda x: -float(x[i_s] or 0))[:20]:
            print(f"  {float(x[i_s]) / tot * 100:5.1f}%  {x[0][-5:]}  {x[i_src][:90]}")


if __name__ == "__main__":
    main()
