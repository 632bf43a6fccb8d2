"""Run bench.py with the given extra args and print a one-line summary."""
import json, subprocess, sys
out = subprocess.run([sys.executable, "bench.py", "--steps", "1000", "--warmup", "20", "--no-cpu-baseline",
                      "--no-e2e"] + sys.argv[1:], capture_output=True, text=True)
if out.returncode:
    print(out.stderr[-2000:]); sys.exit(1)
d = json.loads(out.stdout.strip().splitlines()[-1])
ph = d.get("roofline", {}).get("phases", {})
print(sys.argv[1:], round(d["value"] / 1e6, 2), "M samples/s", round(d["ms_per_step"] * 1e3, 1), "us",
      d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: v for k, v in ph.items() if k != "source"})
