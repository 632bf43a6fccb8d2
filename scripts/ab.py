"""Interleaved A/B of environment knobs on the default bench (developer):
python scripts/ab.py ROUNDS 'A=1' 'GEIG_X=1' ...  -> median us/step per config."""
import json, os, statistics, subprocess, sys
rounds = int(sys.argv[1])
cfgs = sys.argv[2:]
res = {c: [] for c in cfgs}
for r in range(rounds):
    for c in cfgs:
        env = dict(os.environ)
        for kv in c.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "bench.py", "--steps", "2000", "--warmup", "20", "--spinup", "0.3",
                              "--no-cpu-baseline", "--no-e2e"], env=env, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[c].append(d["ms_per_step"] * 1e3)
            print(f"  round {r} {c:40s} {d['ms_per_step']*1e3:6.2f} us  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}",
                  flush=True)
        except Exception:
            print("FAILED", c, out.stderr[-800:], flush=True)
for c in cfgs:
    v = res[c]
    if v:
        print(f"{c:40s} median {statistics.median(v):6.2f} us  min {min(v):6.2f}  (n={len(v)})")
