"""Aggregate ncu SASS-level samples/instructions per CUDA source line.

usage: python tools/ncu_lines.py <report.ncu-rep> <lib.so> [top]
(STALL=stall_long_sb ranks lines by one stall reason instead of all samples;
SECTION=<mangled-name substring> picks the kernel, e.g. gs_sim_kernel_xl)
Maps each SASS offset to its innermost source line via `nvdisasm -g`.
"""
import collections, csv, glob, os, re, subprocess, sys, tempfile

rep, so = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cubin = max(glob.glob(os.path.join(tmp, "*.cubin")), key=os.path.getsize)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
# offsets restart in every kernel's .text section: keep the one profiled
# (SECTION=substring of its mangled name; default the smallest per-warp class)
want = os.environ.get("SECTION", "HotILi64ELi12ELi4E")
insec = False
for l in dis.splitlines():
    if re.match(r"\s*\.section\s+\.text\.", l):
        insec = want in l
        continue
    if not insec:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()[1:]))
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
base = min(int(r[ix["Address"]], 16) for r in data)
samp = collections.Counter(); inst = collections.Counter()
tot = 0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    key = line_of.get(off, "?")
    s = int(r[ix[os.environ.get("STALL", "Warp Stall Sampling (All Samples)")]] or 0)
    samp[key] += s; tot += s
    inst[key] += int(r[ix["Instructions Executed"]] or 0)
itot = sum(inst.values())
print(f"samples {tot}  warp-insts {itot}")
srcs = {}
for key, s in samp.most_common(top):
    f, ln = key.rsplit(":", 1) if ":" in key else (key, "0")
    path = [p for p in glob.glob(f"/root/repo/paper_2309_00558_b200/csrc/{f}")]
    text = ""
    if path:
        srcs.setdefault(f, open(path[0]).read().splitlines())
        text = srcs[f][int(ln) - 1].strip()[:70]
    print(f"{s*100/tot:5.1f}% samp {inst[key]*100/itot:5.1f}% inst  {key:22s} {text}")
