"""Group ncu per-instruction metrics of a kernel into source regions (dev tool).
usage: ncu_regions.py report kernel-substring"""
import collections, csv, re, subprocess, sys
rep, ksub = sys.argv[1], sys.argv[2]
REG = [("rg_render.cu", 114, 206, "fetch"), ("rg_render.cu", 207, 260, "setup_pair+color"),
       ("rg_render.cu", 267, 299, "eval_range"), ("rg_render.cu", 300, 340, "grad_range"),
       ("rg_render.cu", 341, 471, "scatter"), ("rg_render.cu", 576, 612, "expire"),
       ("rg_render.cu", 613, 640, "refill"), ("rg_render.cu", 641, 692, "slab+eval loop"),
       ("rg_render.cu", 693, 760, "composite"), ("rg_render.cu", 761, 790, "bwd tail"),
       ("rg_render.cu", 512, 575, "ray setup"), ("rg_internal.cuh", 120, 150, "isect_exact"),
       ("rg_internal.cuh", 150, 170, "offset_at"), ("rg_render.cu", 94, 113, "box_t")]
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
