"""A/B timing of compile-time variants on C1 (dev tool), medians over repeats:
  python tools/ab.py "" "RG_COLLAPSE_BLOCKS=4" "RG_COLLAPSE_OPEN=2" ...
Each argument is an RG_DEFINES string ("" = the default build); an argument
starting with "env:" sets an environment variable for the default build instead
(e.g. "env:RG_NO_GRAPH=1").  Per variant: 3 runs of tools/quick_time.py blender
--nostats --iters 5, the last 3 iterations of each -> median build / fwd / bwd ms.
Rebuilds the default at the end."""
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(defs):
    env = dict(os.environ, RG_DEFINES=defs)
    return subprocess.run([sys.executable, "paper_2408_03356_b200/build.py", "--force"], cwd=ROOT,
                          env=env, capture_output=True).returncode == 0


def main():
    for v in sys.argv[1:]:
        env = dict(os.environ)
        if v.startswith("env:"):
            k, val = v[4:].split("=", 1)
            env[k] = val
            ok = build("")
        else:
            ok = build(v)
        if not ok:
            print(f"variant [{v}] build failed", flush=True)
            continue
        vals = {"build": [], "fwd": [], "bwd": []}
        for _ in range(3):
            out = subprocess.run([sys.executable, "tools/quick_time.py", "blender", "--nostats",
                                  "--iters", "5"], cwd=ROOT, env=env, capture_output=True,
                                 text=True, timeout=600).stdout
            for line in out.splitlines():
                m = re.search(r"it([2-4]):.*build ([\d.]+) ms\s+fwd ([\d.]+) ms.*bwd ([\d.]+) ms", line)
                if m:
                    vals["build"].append(float(m.group(2)))
                    vals["fwd"].append(float(m.group(3)))
                    vals["bwd"].append(float(m.group(4)))
        med = {k: statistics.median(x) if x else float("nan") for k, x in vals.items()}
        print(f"variant [{v}] median of {len(vals['fwd'])}: build {med['build']:.3f} ms  "
              f"fwd {med['fwd']:.3f} ms  bwd {med['bwd']:.3f} ms  "
              f"sum {sum(med.values()):.3f} ms", flush=True)
    build("")


if __name__ == "__main__":
    main()
