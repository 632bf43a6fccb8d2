"""Mutation probes of the oracle's pins (CPU, ~1-2 min).

Each mutant is a plausible one-token mistake in oracle/ (a dropped term, a
wrong operand, a sign); it is applied to a scratch copy of the repo and the
`-m "not gpu"` oracle pins run against it.  Every mutant must make at least
one pin fail — a mutant that survives marks an unpinned part of the oracle.
Usage: python scripts/oracle_mutants.py [name substring]   (exit 1 if any mutant survives)
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTANTS = [
    ("[By]_j from B_t v_j instead of [Bv]_j", "oracle/game.py", "byj = AUX[j] / den            # [By]_j",
     "byj = BV[j] / den            # [By]_j"),
    ("Alg.3 z-gradient without the chain factor", "oracle/game.py",
     "return (float(V[i] @ AUX[i]) - br) * br * (np.log(nu) - np.log(rho)) * s * (1 - s)",
     "return (float(V[i] @ AUX[i]) - br) * br"),
    ("clip on |<v,[Bv]>|", "oracle/game.py", "max(float(v_j @ aux_j), rho)", "max(abs(float(v_j @ aux_j)), rho)"),
    ("clip at 0 instead of rho", "oracle/game.py", "max(float(v_j @ aux_j), rho)", "max(float(v_j @ aux_j), 0.0)"),
    ("A y_j without the denominator", "oracle/game.py", "a_yj = AV[j] / den            # A_t y_j",
     "a_yj = AV[j]                  # A_t y_j"),
    ("rewards sign", "oracle/game.py", "rewards = (vi @ bvi) * avi - (vi @ avi) * bvi\n    penalties = np.zeros_like(vi)\n    for j in range(i):\n        den = clip",
     "rewards = (vi @ avi) * bvi - (vi @ bvi) * avi\n    penalties = np.zeros_like(vi)\n    for j in range(i):\n        den = clip"),
    ("penalty second term on A_t v_i", "oracle/game.py",
     "penalties += (vi @ a_yj) * ((vi @ bvi) * byj - (vi @ byj) * bvi)\n    return rewards - penalties\n\n\ndef aux_direction",
     "penalties += (vi @ a_yj) * ((vi @ bvi) * byj - (vi @ byj) * avi)\n    return rewards - penalties\n\n\ndef aux_direction"),
    ("penalty sum over j <= i", "oracle/game.py", "    for j in range(i):\n        den = clip_denominator",
     "    for j in range(i + 1):\n        den = clip_denominator"),
    ("aux direction sign", "oracle/game.py", "return BV[i] - AUX[i]", "return AUX[i] - BV[i]"),
    ("no sphere retraction", "oracle/game.py",
     "        V_new[i] = vp / np.linalg.norm(vp)\n        AUX_new[i] = AUX[i] + gamma * gbv\n    return V_new, AUX_new\n",
     "        V_new[i] = vp\n        AUX_new[i] = AUX[i] + gamma * gbv\n    return V_new, AUX_new\n"),
    ("bracket decreasing in z", "oracle/game.py", "(np.log(nu) - np.log(rho)) * _sigmoid(z)))",
     "(np.log(nu) - np.log(rho)) * _sigmoid(-z)))"),
    ("Alg.3 [By]_j from B_t v_j", "oracle/game.py", "byj = AUX[j] / den\n        penalties +=",
     "byj = BV[j] / den\n        penalties +="),
    ("A_t from the B half of the rows", "oracle/estimators.py", "av = np.concatenate([x1.T @ (y1 @ vy), y1.T @ (x1 @ vx)], axis=0) / h",
     "av = np.concatenate([x1.T @ (y2 @ vy), y1.T @ (x2 @ vx)], axis=0) / h"),
    ("B_t cross-view", "oracle/estimators.py", "bv = np.concatenate([x2.T @ (x2 @ vx), y2.T @ (y2 @ vy)], axis=0) / h",
     "bv = np.concatenate([x2.T @ (y2 @ vy), y2.T @ (x2 @ vx)], axis=0) / h"),
    ("Adam without bias correction", "oracle/game.py", "mh = m / (1 - b1 ** t)", "mh = m"),
    ("Alg.1 parent normalised by the Euclidean norm", "oracle/game.py",
     "yj = V[j] / np.sqrt(V[j] @ b @ V[j])", "yj = V[j] / np.linalg.norm(V[j])"),
]


def main():
    tests = [os.path.join("tests", f) for f in sorted(os.listdir(os.path.join(ROOT, "tests")))
             if f.startswith("test_oracle_")]
    survived = []
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for name, rel, old, new in MUTANTS:
        if only not in name:
            continue
        with tempfile.TemporaryDirectory() as tmp:
            for part in ("oracle", "synth", "tests"):
                shutil.copytree(os.path.join(ROOT, part), os.path.join(tmp, part))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            path = os.path.join(tmp, rel)
            src = open(path).read()
            if src.count(old) != 1:
                print(f"?? {name}: pattern found {src.count(old)} times")
                survived.append(name)
                continue
            open(path, "w").write(src.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", *tests],
                               cwd=tmp, capture_output=True, text=True)
            killed = r.returncode != 0
            first = next((l for l in r.stdout.splitlines() if l.startswith("FAILED")), "")
            print(f"{'killed ' if killed else 'SURVIVED'} {name}  {first}")
            if not killed:
                survived.append(name)
    n = sum(1 for m in MUTANTS if only in m[0])
    print(f"{n - len(survived)}/{n} mutants killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
