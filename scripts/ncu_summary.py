"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python scripts/ncu_summary.py <tag> <launches.csv> <prof.ncu-rep> [config/ordering]

Writes profiles/<tag>_launches.md (per-kernel device time from the
gpu__time_duration launch list), profiles/<tag>_ncu_full.md (key metrics of
the --set full capture) and merges per-launch DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (DMMA)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("feti::", "")


def launches(path, metric="gpu__time_duration.sum", scale=1e-6):
    """Per-kernel list of one metric over every launch of a --metrics CSV
    (durations in ms by default; several metrics may share the file)."""
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        # the capture's -k filter keeps our kernels only (names may or may not
        # carry the feti:: namespace depending on the ncu version)
        if "Kernel Name" not in d or d.get("Metric Name", metric) != metric:
            continue
        agg.setdefault(short(d["Kernel Name"]), []).append(float(d["Metric Value"].replace(",", "")) * scale)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, label in KEYS:
            if k in hdr:
                d[label] = (r[hdr.index(k)], units[hdr.index(k)])
        res.append(d)
    return res


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    try:
        return float(v) * scale
    except ValueError:
        return None


def main():
    tag, lpath, fpath = sys.argv[1:4]
    key = sys.argv[4] if len(sys.argv) > 4 else "c3/rcm"
    os.makedirs(PROF, exist_ok=True)
    agg = launches(lpath)
    tot = sum(sum(v) for v in agg.values())
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as fh:
        fh.write(f"# {tag}: launch list (ncu gpu__time_duration.sum, --clock-control none)\n\n")
        fh.write("Cold-cache, serialised per-launch device times: compare SHARES, not absolutes.\n\n")
        fh.write("| kernel | launches | mean ms | total ms | share |\n|---|---|---|---|---|\n")
        for k, v in agg.items():
            fh.write(f"| {k} | {len(v)} | {sum(v) / len(v):.4f} | {sum(v):.3f} | {sum(v) / tot:.1%} |\n")
    res = full(fpath)
    with open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w") as fh:
        fh.write(f"# {tag}: ncu --set full (one launch per kernel)\n\n")
        labels = [label for _, label in KEYS]
        fh.write("| kernel | " + " | ".join(labels) + " |\n|---|" + "---|" * len(labels) + "\n")
        for d in res:
            fh.write(f"| {d['kernel']} | " + " | ".join(
                f"{d[l][0]} {d[l][1]}".strip() if l in d else "" for l in labels) + " |\n")
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    ent = traffic.setdefault(key, {})
    for d in res:
        if "dram read" in d and "dram write" in d:
            rb, wb = to_bytes(*d["dram read"]), to_bytes(*d["dram write"])
            if rb is not None and wb is not None:
                ent[d["kernel"]] = rb + wb
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print(open(os.path.join(PROF, f"{tag}_launches.md")).read())
    print(open(os.path.join(PROF, f"{tag}_ncu_full.md")).read())


if __name__ == "__main__":
    main()
