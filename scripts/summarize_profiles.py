"""Summarise an ncu launch list and a full capture into profiles/ (developer tool)."""
import csv, json, subprocess, sys, collections

def launch_list(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr = r; start = i + 1; break
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        u = u.strip().lower()
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        agg.setdefault(r[ki].split("(")[0].strip(), []).append(v)
    return agg

def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for w in want:
            if w in hdr:
                d[w] = r[hdr.index(w)] + " " + units[hdr.index(w)]
        res.append(d)
    return res

if __name__ == "__main__":
    tag = sys.argv[1]
    ll = launch_list(sys.argv[2])
    fc = full_capture(sys.argv[3])
    lines = [f"# ncu summary — {tag}", "", "## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
             "| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
    ours = {k: v for k, v in ll.items() if "geig::" in k or "tc::" in k}
    tot = sum(sum(v) for v in ours.values()) or 1.0
    lines[-2] = "| kernel | launches | mean us | share of this repo's kernel time |"
    for k, v in ll.items():
        share = f"{sum(v)/tot:.3f}" if k in ours else "(input synthesis, untimed)"
        lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v)/len(v):.1f} | {share} |")
    lines += ["", "## Full capture (--set full), per launch", ""]
    for d in fc:
        lines.append(f"### `{d['kernel'][:100]}`")
        for k, v in d.items():
            if k != "kernel":
                lines.append(f"- {k}: {v}")
        lines.append("")
    open(f"profiles/{tag}_ncu_summary.md", "w").write("\n".join(lines))
    json.dump({"launch_list": {k: v for k, v in ll.items()}, "full": fc}, open(f"profiles/{tag}_ncu.json", "w"), indent=1)
    print("\n".join(lines))
