"""Per-function (source-level) samples / instructions of an ncu report.

usage: python tools/ncu_funcs.py <report.ncu-rep> <lib.so> [kernel-substring] [top]
Each SASS instruction is attributed to its innermost source line (nvdisasm -g),
then to the enclosing function of that line in csrc/.
"""
import collections, csv, glob, os, re, subprocess, sys, tempfile

rep, so = sys.argv[1], sys.argv[2]
kname = sys.argv[3] if len(sys.argv) > 3 else "HotILi64"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2309_00558_b200", "csrc")
fn_of = {}
for path in glob.glob(os.path.join(CSRC, "*")):
    cur = "?"
    for i, l in enumerate(open(path).read().splitlines(), 1):
        m = re.match(r"^(?:template.*>\s*)?(?:__device__|__global__|static|inline|extern|__host__)[^;(]*?(\w+)\(", l)
        if m and not l.startswith("//"):
            cur = m.group(1)
        fn_of[(os.path.basename(path), i)] = cur
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = max(glob.glob(tmp + "/*.cubin"), key=os.path.getsize)
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
secs = re.split(r"\n\s*\.section\s+\.text\.", dis)
dis = [s for s in secs if s.startswith("_ZN2gs") and "gs_sim_kernel" in s.split(",")[0] and kname in s.split(",")[0]][0]
line_of, cur = {}, None
for l in dis.splitlines():
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()[1:]))
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
base = min(int(r[ix["Address"]], 16) for r in data)
S, I = collections.Counter(), collections.Counter()
tot = itot = 0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    key = line_of.get(off)
    name = fn_of.get(key, key[0] if key else "?") if key else "?"
    S[name] += s; I[name] += n; tot += s; itot += n
print(f"samples {tot} warp-insts {itot}")
for k, v in S.most_common(top):
    print(f"{k:28s} samp {v*100/tot:5.1f}%  inst {I[k]*100/itot:5.1f}%")
