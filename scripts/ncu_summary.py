"""Summarise ncu captures of one decode step into profiles/.

  python scripts/ncu_summary.py <cfg> <launches.csv> <full.ncu-rep> <out_dir>

launches.csv: `ncu --metrics gpu__time_duration.sum --csv` over exactly one decode
step (cold-cache, serialised: compare SHARES, not absolute times); full.ncu-rep:
`ncu --set full` of one layer's GEMMs + attention. Writes launch_summary_<cfg>.csv,
ncu_full_<cfg>.json and updates profiles/ncu_traffic.json (DRAM bytes per launch,
the `traffic` field of bench.py's roofline object).
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def classify(names):
    """Kernel names of one step in launch order -> bench.py kernel classes."""
    out, after_attn = [], False
    for n in names:
        if "embed_norm" in n:
            out.append("embed_norm")
        elif "attn_decode" in n:
            out.append("attention")
            after_attn = True
        elif "attn_combine" in n:
            out.append("attn_combine")
        elif "gemm_chain" in n:
            out.append("gemm_chain")
        elif "argmax" in n:
            out.append("argmax")
        elif "gemm_kernel<2" in n:
            out.append("gemm_qkv_rope_kv")
        elif "gemm_kernel<3" in n:
            out.append("gemm_gate_up_swiglu")
        elif "gemm_kernel<4" in n:
            out.append("gemm_lm_head_argmax")
        elif "gemm_kernel<1" in n:
            out.append("gemm_o_resid_norm" if after_attn else "gemm_down_resid_norm")
            after_attn = False
        else:
            out.append(n)
    return out


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    hdr = next(r for r in csv.reader(open(path)) if r and r[0] == "ID")
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    names = [r[i_name] for r in rows]
    ts = [float(r[i_val].replace(",", "")) / 1e3 for r in rows]  # ns -> us
    return names, ts


def main():
    cfg, lpath, rep, out = sys.argv[1:5]
    os.makedirs(out, exist_ok=True)
    names, ts = launches(lpath)
    cls = classify(names)
    agg = OrderedDict()
    for c, t in zip(cls, ts):
        a = agg.setdefault(c, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(ts)
    with open(os.path.join(out, f"launch_summary_{cfg}.csv"), "w") as f:
        f.write(f"# ncu launch list, {cfg}, one decode step ({len(ts)} launches, {total:.1f} us serialised)\n")
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)\n")
        f.write("kernel,launches,total_us,avg_us,share\n")
        for c, (k, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{c},{k},{t:.1f},{t / k:.2f},{t / total:.3f}\n")
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
               "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
               "launch__cluster_dim_x", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kern = []
    for r in data:
        d = {h: v for h, v in zip(hdr, r) if h in metrics or h == "Kernel Name"}
        kern.append(d)
    knames = classify([k["Kernel Name"] for k in kern])
    for k, c in zip(kern, knames):
        k["class"] = c
    with open(os.path.join(out, f"ncu_full_{cfg}.json"), "w") as f:
        json.dump({"command": f"ncu --set full --clock-control none --import-source on (one layer of {cfg})",
                   "units": {h: u for h, u in zip(hdr, units) if h in metrics}, "kernels": kern}, f, indent=1)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    unit = {h: u for h, u in zip(hdr, units)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    t = {}
    for k in kern:
        rb = float(k["dram__bytes_read.sum"]) * scale[unit["dram__bytes_read.sum"]]
        wb = float(k["dram__bytes_write.sum"]) * scale[unit["dram__bytes_write.sum"]]
        t[k["class"]] = rb + wb
    traffic[cfg] = t
    traffic["source"] = "profiles/<round>/ncu_full_<cfg>.json: dram__bytes_read.sum + dram__bytes_write.sum per launch"
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(open(os.path.join(out, f"launch_summary_{cfg}.csv")).read())
    print(json.dumps(t, indent=1))


if __name__ == "__main__":
    main()
