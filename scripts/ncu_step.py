"""Per-step launch list with DRAM traffic from an ncu --metrics CSV.

    python scripts/ncu_step.py <tag> <launches.csv> <steps> [config/ordering]

The CSV is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`
over `scripts/factor_bench.py <cfg> 1` (every launch of <steps> preprocesses).  Writes
profiles/<tag>_launches.md (time share + DRAM bytes per kernel and per step) and merges the
step's total DRAM traffic into profiles/ncu_traffic.json ("step (fused graph, per step)"),
which bench.py reports as roofline.traffic.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import PROF, launches  # noqa: E402


def main():
    tag, path, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
    key = sys.argv[4] if len(sys.argv) > 4 else "c3/sparse"
    t = launches(path)
    rd = launches(path, "dram__bytes_read.sum", 1.0)
    wr = launches(path, "dram__bytes_write.sum", 1.0)
    tot = sum(sum(v) for v in t.values())
    step_bytes = 0.0
    lines = [f"# {tag}: launch list of {steps} steps (ncu, --clock-control none)\n",
             "Cold-cache, serialised per-launch device times: compare SHARES, not absolutes.  DRAM bytes are",
             "per step (read + write, summed over the kernel's launches / steps).\n",
             "| kernel | launches / step | mean ms | share of time | DRAM GB / step |", "|---|---|---|---|---|"]
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        b = (sum(rd.get(k, [])) + sum(wr.get(k, []))) / steps
        step_bytes += b
        lines.append(f"| {k} | {len(v) / steps:.0f} | {sum(v) / len(v):.4f} | {sum(v) / tot:.1%} | {b / 1e9:.2f} |")
    lines.append(f"\nStep total: {step_bytes / 1e9:.2f} GB DRAM, {tot / steps:.1f} ms serialised launch time.")
    out = os.path.join(PROF, f"{tag}_launches.md")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic.setdefault(key, {})["step (fused graph, per step)"] = step_bytes
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
