"""Per-source-line samples/instructions of an ncu report, split into the
quantum-step subroutine (hot_steps) and everything else.

usage: python tools/ncu_regions.py <report.ncu-rep> <lib.so> [kernel-substring] [top]
"""
import collections, csv, glob, os, re, subprocess, sys, tempfile

rep, so = sys.argv[1], sys.argv[2]
kname = sys.argv[3] if len(sys.argv) > 3 else "HotILi64"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = glob.glob(tmp + "/*.cubin")[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
secs = re.split(r"\n\s*\.section\s+\.text\.", dis)
dis = [s for s in secs if s.startswith("_ZN2gs") and "gs_sim_kernel" in s.split(",")[0] and kname in s.split(",")[0]][0]
line_of, op_of, cur = {}, {}, None
for l in dis.splitlines():
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
        op_of[int(m.group(1), 16)] = m.group(2)
# subroutines: targets of CALL.REL (nvdisasm prints labels; find RET-delimited blocks after the main RET/EXIT)
addrs = sorted(op_of)
rets = [a for a in addrs if op_of[a].split()[0].lstrip("@!P0123456789 ").startswith("RET")]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()[1:]))
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
base = min(int(r[ix["Address"]], 16) for r in data)
# hot_steps = the largest RET-delimited block that contains gs_hot.cuh:hot_step lines
blocks = []
prev = None
for r_ in rets:
    lo = prev + 16 if prev is not None else None
    blocks.append((lo, r_))
    prev = r_
def region(off):
    for lo, hi in blocks[1:]:
        if lo <= off <= hi:
            return f"sub@{lo:x}"
    return "main"
S, I = collections.Counter(), collections.Counter()
LS, LI = collections.defaultdict(collections.Counter), collections.defaultdict(collections.Counter)
tot = itot = 0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    g = region(off)
    S[g] += s; I[g] += n; tot += s; itot += n
    LS[g][line_of.get(off, "?")] += s; LI[g][line_of.get(off, "?")] += n
srcs = {}
def text(key):
    f, ln = key.rsplit(":", 1) if ":" in key else (key, "0")
    p = glob.glob(f"/root/repo/paper_2309_00558_b200/csrc/{f}")
    if not p:
        return ""
    srcs.setdefault(f, open(p[0]).read().splitlines())
    return srcs[f][int(ln) - 1].strip()[:64]
print(f"samples {tot} warp-insts {itot}")
for g in sorted(S, key=lambda k: -S[k]):
    print(f"== {g}: samples {S[g]*100/tot:.1f}%  inst {I[g]*100/itot:.1f}%  size {sum(1 for a in addrs if region(a)==g)} instr")
    for key, s in LS[g].most_common(top):
        print(f"   {s*100/tot:5.1f}% samp {LI[g][key]*100/itot:5.1f}% inst  {key:22s} {text(key)}")
