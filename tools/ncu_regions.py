"""Group ncu per-instruction metrics of a kernel into source regions (dev tool).
usage: ncu_regions.py report kernel-substring [--rev GIT_REV]
--rev reads the sources of the profiled build from git (line numbers drift)"""
import collections, csv, re, subprocess, sys
REV = None
if "--rev" in sys.argv:
    i = sys.argv.index("--rev"); REV = sys.argv[i + 1]; del sys.argv[i:i + 2]
rep, ksub = sys.argv[1], sys.argv[2]
import os
CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2408_03356_b200", "csrc")
def auto_regions():
    """function definitions and '// ---- label' markers delimit regions"""
    reg = []
    for fn in ("rg_render.cu", "rg_internal.cuh"):
        if REV:
            lines = subprocess.run(["git", "show", f"{REV}:paper_2408_03356_b200/csrc/{fn}"],
                                   capture_output=True, text=True, check=True,
                                   cwd=os.path.dirname(CSRC)).stdout.splitlines()
        else:
            lines = open(os.path.join(CSRC, fn)).read().splitlines()
        marks = []
        for i, l in enumerate(lines, 1):
            m = re.match(r"^(?:template.*\n)?__(?:device|global)__.*?\b(\w+)\s*\(", l)
            if m and not l.strip().endswith(";"):
                marks.append((i, m.group(1)))
            m2 = re.match(r"^\s*// ---- (\w[\w ]*)", l)
            if m2:
                marks.append((i, "k:" + m2.group(1)[:20]))
        for k, (a, name) in enumerate(marks):
            b = marks[k + 1][0] - 1 if k + 1 < len(marks) else len(lines)
            reg.append((fn, a, b, name))
    return reg
REG = auto_regions()
def page(view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
amap = {}; fn = path = None; cur = None
for r in page("cuda,sass"):
    if not r: continue
    if r[0] == "File Path": path = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": fn = r[1]; continue
    if r[0] == "Line No": continue
    if r[0]: cur = (path, int(r[0]))
    elif len(r) > 2 and r[2].startswith("0x"): amap[(fn, r[2])] = cur
def region(fl):
    if fl is None: return "?"
    f, l = fl
    for ff, a, b, name in REG:
        if f == ff and a <= l <= b: return name
    return f"{f}:other"
kern = None; hdr = None
agg = collections.defaultdict(lambda: collections.Counter())
for r in page("sass"):
    if not r: continue
    if r[0] == "Kernel Name": kern = r[1]; hdr = None; continue
    if hdr is None:
        if "Instructions Executed" in r: hdr = r
        continue
    if ksub not in kern: continue
    d = dict(zip(hdr, r))
    reg = region(amap.get((kern, d["Address"])))
    for m in ("Instructions Executed", "Warp Stall Sampling (All Samples)", "Thread Instructions Executed"):
        try: agg[m][reg] += float(d.get(m) or 0)
        except ValueError: pass
ins = agg["Instructions Executed"]; st = agg["Warp Stall Sampling (All Samples)"]; th = agg["Thread Instructions Executed"]
ti, ts = sum(ins.values()) or 1, sum(st.values()) or 1
print(f"{'region':22s} {'inst%':>6s} {'stall%':>7s} {'lanes/inst':>10s}  (total warp-inst {ti/1e9:.2f} G)")
for k, v in sorted(ins.items(), key=lambda x: -st[x[0]]):
    print(f"{k:22s} {100*v/ti:6.1f} {100*st[k]/ts:7.1f} {th[k]/max(v,1):10.1f}")
