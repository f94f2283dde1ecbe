"""Summarise ncu captures into markdown for profiles/ (run here, no GPU):

  python tools/ncu_summary.py --rep gpurun_out/prof_ar_n1.ncu-rep --rep ... \
      --launches gpurun_out/launches.csv --out profiles/round1_ncu.md
"""
import argparse
import collections
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki]
        if any(k in name for k in ("coll_kernel", "local_copy_kernel", "nvls_kernel", "a2a_tma_kernel")):
            key = "lagom collectives (sm_100a)"
        elif "fill_kernel" in name or "timestamp_kernel" in name:
            key = "lagom fill / timestamp kernels (setup only)"
        elif "cudnn" in name or "sdpa" in name:
            key = "cuDNN SDPA attention (victims)"
        else:
            key = "cuBLASLt GEMMs (victims)"
        tot[key] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[key] += 1
    return tot, cnt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--label", action="append", default=[])
    ap.add_argument("--launches", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="round 2")
    a = ap.parse_args()
    md = [f"# ncu summaries ({a.title})", ""]
    for i, rep in enumerate(a.rep):
        label = a.label[i] if i < len(a.label) else rep
        md += [f"## {label}", "", f"source: `{rep}` (`ncu --set full --clock-control none`)", ""]
        for hdr, units, r in raw(rep):
            md += [f"kernel: `{r[hdr.index('Kernel Name')]}`", "", "| metric | value |", "|---|---|"]
            for m, nice in METRICS:
                if m in hdr:
                    j = hdr.index(m)
                    md.append(f"| {nice} (`{m}`) | {r[j]} {units[j]} |")
            md.append("")
    if a.launches:
        tot, cnt = launches(a.launches)
        T = sum(tot.values())
        md += ["## launch list shares", "", f"source: `{a.launches}` (`--metrics gpu__time_duration.sum`, "
               "cold-cache and serialised: compare shares, not absolutes)", "",
               "| kernel class | launches | total us | share |", "|---|---|---|---|"]
        for k in sorted(tot, key=tot.get, reverse=True):
            md.append(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / T:.3f} |")
        md.append("")
    with open(a.out, "w") as f:
        f.write("\n".join(md))


if __name__ == "__main__":
    main()
