"""Developer tool: aggregate an ncu --set full source page (SASS csv) of the
fused step kernel by CUDA source line using the cubin's line table.
usage: python scripts/ncu_lines.py <report.ncu-rep> <file.cuh> <line_lo> <line_hi>"""
import csv, io, re, subprocess, sys, tempfile, os
rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
kern = os.environ.get("KERN", "_ZN4geig2tc15cca_step_kernelILi2EEEvNS0_9FusedMapsENS0_11FusedParamsE")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
ix = {n: i for i, n in enumerate(h)}
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath("paper_2206_04993_b200/libgeig.so")], cwd=td,
                   capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(td, cub)], capture_output=True,
                          text=True).stdout.split("\n")
start = [i for i, l in enumerate(sass) if l.startswith(".text." + kern + ":")][0]
cur = None; m = {}
for l in sass[start + 1:]:
    if l.startswith(".text.") or l.startswith(".section"):
        break
    mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if mm:
        cur = (mm.group(1).split("/")[-1], int(mm.group(2))); continue
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mo and cur:
        m[int(mo.group(1), 16)] = cur
base = int(data[0][0], 16)
stall = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
agg = {}
tot = 0.0
for r in data:
    tot += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    key = m.get(int(r[0], 16) - base, ("?", 0))
    if key[0] != fname or not (lo <= key[1] <= hi):
        continue
    a = agg.setdefault(key[1], {"n": 0.0, "wf": 0.0, "wfi": 0.0, **{n: 0.0 for n in stall}})
    a["n"] += float(r[ix["Instructions Executed"]] or 0)
    a["wf"] += float(r[ix["L1 Wavefronts Shared"]] or 0)
    a["wfi"] += float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
    for n in stall:
        a[n] += float(r[ix[n]] or 0)
print(f"total samples {tot:.0f}")
for ln in sorted(agg):
    a = agg[ln]
    t = sum(a[n] for n in stall)
    if t < 3 and a["wf"] == 0:
        continue
    top = sorted(((a[n], n) for n in stall if a[n] > 0), reverse=True)[:4]
    print(f"{ln:5d} samples {t:6.0f} ({100*t/tot:4.1f}%) instr {a['n']:9.0f} smem wf {a['wf']:8.0f}/{a['wfi']:8.0f} ",
          [(n[6:], int(v)) for v, n in top])
