"""Summarise the ncu captures of one profiling round into profiles/ (tracked):
  python profiles/summarize.py r01
reads gpurun_out/launches_<tag>.csv and gpurun_out/<kernel>_<tag>.ncu-rep and
writes profiles/ncu_<tag>.md, profiles/ncu_<tag>.json and (for bench.py's
roofline "traffic" key) profiles/xterm_traffic.json."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
KERNELS = ["k_xterm", "k_moments_i8", "k_texthist", "k_hist_contract", "k_finalize_i8", "k_finalize_rows",
           "k_finalize_maxima_c5"]
KERNELS_C3 = ["k_xterm_c3", "k_split_f32_c3"]  # float path (C3 bench step), tools/ncu_r02.sh
METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-3),  # reported in us by default -> ms below
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "tensor_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", None),
    "imma_active_pct": ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "hmma_active_pct": ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    "smem_lsu_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", None),
    "smem_tc_wavefronts": ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", None),
    "l1tex_pct_peak": ("l1tex__throughput.avg.pct_of_peak_sustained_active", None),
    "l2_pct_peak": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "l2_to_sm_bytes": ("l1tex__m_xbar2l1tex_read_bytes.sum", None),
    "sm_cycles": ("sm__cycles_elapsed.avg", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
              "second": 1e3, "s": 1e3}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def kernel_summary(rep):
    d = raw(rep)
    out = {}
    for key, (m, _) in METRICS.items():
        if m not in d:
            continue
        v, u = d[m]
        x = num(v)
        if x is None:
            continue
        if key == "duration_ms":
            x *= UNIT_SCALE.get(u, 1e-3)
        elif u in UNIT_SCALE and "byte" in u:
            x *= UNIT_SCALE[u]
        out[key] = x
    return out


def launches(tag, prefix="launches"):
    p = os.path.join(OUT, f"{prefix}_{tag}.csv")
    if not os.path.exists(p):
        return {}
    txt = open(p).read()
    lines = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in csv.DictReader(io.StringIO(lines)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("::")[-1]
        scale = UNIT_SCALE.get(r.get("Metric Unit", "nsecond"), 1e-6)
        tot[name] += num(r["Metric Value"]) * scale
        cnt[name] += 1
    s = sum(tot.values()) or 1.0
    return {k: {"launches": cnt[k], "ms_total": tot[k], "share": tot[k] / s} for k in sorted(tot, key=lambda k: -tot[k])}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    res = {"tag": tag, "launch_list": launches(tag), "kernels": {}}
    for k in KERNELS + KERNELS_C3:
        rep = os.path.join(OUT, f"{k}_{tag}.ncu-rep")
        if os.path.exists(rep):
            res["kernels"][k] = kernel_summary(rep)
    res["launch_list_c3"] = launches(tag, "launches_c3")
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.json"), "w") as f:
        json.dump(res, f, indent=1)
    lines = [f"# ncu summary, {tag} (C4: 1.5M x 5000 int8, one bench step)", "",
             "Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised):", "",
             "| kernel | launches | ms (sum) | share |", "|---|---|---|---|"]
    for k, v in res["launch_list"].items():
        lines.append(f"| {k} | {v['launches']} | {v['ms_total']:.3f} | {v['share'] * 100:.1f}% |")
    lines += ["", "Full captures (`--set full --clock-control none`, second step):", "",
              "| kernel | ms | DRAM read GB | DRAM write GB | DRAM % | tensor % | issue % | smem LSU wf | smem TC wf | L2->SM GB | L2 % | regs |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, v in res["kernels"].items():
        g = lambda n, sc=1.0, f="{:.2f}": (f.format(v[n] * sc) if n in v else "-")
        lines.append(f"| {k} | {g('duration_ms')} | {g('dram_read_bytes', 1e-9)} | {g('dram_write_bytes', 1e-9)} | "
                     f"{g('dram_pct_peak', 1, '{:.1f}')} | {g('tensor_active_pct', 1, '{:.1f}')} | "
                     f"{g('issue_active_pct', 1, '{:.1f}')} | {g('smem_lsu_wavefronts', 1, '{:.3g}')} | "
                     f"{g('smem_tc_wavefronts', 1, '{:.3g}')} | {g('l2_to_sm_bytes', 1e-9)} | "
                     f"{g('l2_pct_peak', 1, '{:.1f}')} | {g('registers', 1, '{:.0f}')} |")
    if res["launch_list_c3"]:
        lines += ["", "C3 (100K x 5000 float32) launch list:", "", "| kernel | launches | ms (sum) | share |",
                  "|---|---|---|---|"]
        for k, v in res["launch_list_c3"].items():
            lines.append(f"| {k} | {v['launches']} | {v['ms_total']:.3f} | {v['share'] * 100:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    for kname, cfg, fname in (("k_xterm", "C4", "xterm_traffic.json"), ("k_xterm_c3", "C3", "xterm_traffic_C3.json")):
        x = res["kernels"].get(kname)
        if not (x and "dram_read_bytes" in x):
            continue
        with open(os.path.join(ROOT, "profiles", fname), "w") as f:
            ms = x.get("duration_ms")
            cyc = x.get("sm_cycles")
            json.dump({"config": cfg, "n_gpus": 1, "tag": tag,
                       "dram_bytes_per_launch": x["dram_read_bytes"] + x.get("dram_write_bytes", 0.0),
                       "tensor_active_pct": x.get("tensor_active_pct"),
                       "duration_ms": ms,
                       # the kernel's own average SM clock (cycles / duration): nvidia-smi's
                       # coarse samples overstate it under the power cap
                       "sm_mhz": (cyc / (ms * 1e-3) / 1e6) if (cyc and ms) else None,
                       "source": f"ncu --set full capture gpurun_out/{kname}_{tag}.ncu-rep (profiles/ncu_{tag}.md)"}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
