"""Summarise ncu outputs for profiles/ (markdown on stdout).

    python tools/summarize_profiles.py LAUNCHES.csv [REPORT.ncu-rep ...] [--traffic OUT.json]

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` output;
reports: `ncu --set full -o` captures.  `--traffic` writes, per LL kernel
name, the mean DRAM bytes (read + write) per launch from the full captures
(bench.py reads it for roofline.traffic).
"""

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | mean us | share of all GPU time |")
    print("|---|---|---|---|")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k[:70]}` | {n} | {s / n / 1e3:.2f} | {100 * s / tot:.1f}% |")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def full(rep, traffic):
    hdr, body = raw(rep)
    col = {n: i for i, n in enumerate(hdr)}

    def get(r, name, default="-"):
        i = col.get(name)
        return r[i] if i is not None and i < len(r) and r[i] != "" else default

    print(f"\n`{rep.split('/')[-1]}`\n")
    print("| kernel | us | DRAM read MB | DRAM write MB | DRAM % peak | SM active % | warps/SM | regs | grid x block |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in body:
        name = get(r, "Kernel Name")
        short = name.split("(")[0].replace("void ", "")[:48]
        dur = float(get(r, "gpu__time_duration.sum", "0").replace(",", ""))
        rd = float(get(r, "dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(get(r, "dram__bytes_write.sum", "0").replace(",", ""))
        unit = hdr_units.get("dram__bytes_read.sum", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        rd *= scale
        wr *= scale
        dunit = hdr_units.get("gpu__time_duration.sum", "nsecond")
        us = dur * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(dunit, 1.0)
        print(f"| `{short}` | {us:.2f} | {rd / 1e6:.2f} | {wr / 1e6:.2f} | "
              f"{get(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
              f"{get(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
              f"{get(r, 'sm__warps_active.avg.per_cycle_active')} | {get(r, 'launch__registers_per_thread')} | "
              f"{get(r, 'launch__grid_size')} x {get(r, 'launch__block_size')} |")
        for key, pat in (("epb_ll_dispatch", "ll_dispatch_kernel"), ("epb_ll_combine", "ll_combine_kernel")):
            if pat in name:
                traffic.setdefault(key, []).append(rd + wr)


hdr_units = {}


def main():
    args = [a for a in sys.argv[1:]]
    out_traffic = None
    if "--traffic" in args:
        i = args.index("--traffic")
        out_traffic = args[i + 1]
        del args[i:i + 2]
    launches(args[0])
    traffic = {}
    for rep in args[1:]:
        hdr, body = raw(rep)
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr_units.clear()
        hdr_units.update({n: u for n, u in zip(rows[0], rows[1])})
        full(rep, traffic)
    if out_traffic:
        json.dump({k: int(sum(v) / len(v)) for k, v in traffic.items()}, open(out_traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
