"""Summarise ncu outputs into profiles/ (run in the build container).

  python tools/summarize_ncu.py launches gpurun_out/launches.csv profiles/r01_launches.md
  python tools/summarize_ncu.py full gpurun_out/upgate.ncu-rep profiles/r01_upgate.md [flops_per_launch]
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct"]


def launches(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1000.0 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1000.0
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(t for _, t in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / total:.1f}% |")
    open(out, "w").write(f"# ncu launch list (`{path}`)\n\ncold-cache, serialised per-launch times "
                         f"(shares are what matter)\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out, flops=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    lines = ["| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " | unit |",
             "|---|" + "---|" * (len(rows) - 2) + "---|"]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            vals = [r[i] for r in rows[2:]]
            res[k] = vals
            lines.append(f"| {k} | " + " | ".join(vals) + f" | {units[i]} |")
    names = [r[hdr.index("Kernel Name")] for r in rows[2:]] if "Kernel Name" in hdr else []
    txt = f"# ncu --set full: `{path}`\n\nkernels: {names}\n\n" + "\n".join(lines) + "\n"
    if flops:
        t = float(res["gpu__time_duration.sum"][0].replace(",", ""))
        unit = units[hdr.index("gpu__time_duration.sum")]
        sec = t * (1e-9 if unit in ("ns", "nsecond") else 1e-6 if unit in ("us", "usecond") else 1e-3)
        txt += f"\nalgorithmic FLOP per launch {float(flops):.4g} -> {float(flops) / sec / 1e12:.1f} TFLOP/s under ncu\n"
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def nbytes(k):  # each metric carries its own unit
        if k not in hdr:
            return 0.0
        return float(res[k][0].replace(",", "")) * scale.get(units[hdr.index(k)], 1)

    traffic = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    txt += f"\nDRAM traffic per launch (read+write): {traffic:.4g} bytes\n"
    open(out, "w").write(txt)
    print(txt)
    return traffic


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tr = full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
        if len(sys.argv) > 5:
            json.dump({"mlp_up_gate_bytes_per_launch": tr, "source": sys.argv[2]}, open(sys.argv[5], "w"))
