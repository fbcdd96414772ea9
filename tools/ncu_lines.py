"""Aggregate ncu warp-stall samples per CUDA source line (dev tool).
usage: ncu_lines.py report.ncu-rep [kernel-substring] [topN]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]; metric = "Instructions Executed" if "--inst" in sys.argv else "Warp Stall Sampling (All Samples)"
sys.argv=[a for a in sys.argv if a!="--inst"]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
def page(view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
amap = {}; fn = None; path = None; cur = None
for r in page("cuda,sass"):
    if not r: continue
    if r[0] == "File Path": path = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": fn = r[1]; continue
    if r[0] == "Line No": continue
    if r[0]:
        cur = f"{path}:{r[0]} {r[1].strip()[:80]}"
    elif len(r) > 2 and r[2].startswith("0x"):
        amap[(fn, r[2])] = cur
kern = None; hdr = None
per = collections.defaultdict(collections.Counter); stall = collections.defaultdict(collections.Counter)
for r in page("sass"):
    if not r: continue
    if r[0] == "Kernel Name": kern = r[1]; hdr = None; continue
    if hdr is None:
        if "Warp Stall Sampling (All Samples)" in r: hdr = r
        continue
    d = dict(zip(hdr, r))
    if ksub not in kern: continue
    s = float(d.get(metric) or 0)
    per[kern][amap.get((kern, d["Address"]), "?")] += s
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            try: stall[kern][k] += float(d[k] or 0)
            except ValueError: pass
for k in per:
    tot = sum(per[k].values()) or 1
    print("=====", k[:70], "samples", int(tot))
    for l, s in per[k].most_common(top): print(f"{100*s/tot:5.1f}%  {l}")
    print("stalls:", ", ".join(f"{a[6:]} {100*b/tot:.1f}%" for a, b in stall[k].most_common(9)))
