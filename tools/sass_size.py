"""Static SASS size of a kernel attributed to source functions, following
the inline chain (nvdisasm -gi) to the innermost frame that is not a CUDA
header.  usage: python tools/sass_size.py <lib.so> [kernel-substring] [top]"""
import collections, glob, os, re, subprocess, sys, tempfile
so = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else "HotILi64"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
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
cub = glob.glob(tmp + "/*.cubin")[0]
txt = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
secs = re.split(r"\n\s*\.section\s+\.text\.", txt)
sec = [s for s in secs if s.startswith("_ZN2gs13gs_sim_kernel") and kname in s.split(",")[0]][0]
chain, in_chain = [], False
cnt, total = collections.Counter(), 0
for l in sec.split("\n"):
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        if not in_chain:
            chain = []
        in_chain = True
        chain.append((os.path.basename(m.group(1)), int(m.group(2))))
        continue
    in_chain = False
    if re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+", l):
        total += 1
        ours = [fr for fr in chain if fr in fn_of]
        cnt[fn_of[ours[0]] if ours else "?"] += 1
print("total", total)
for k, v in cnt.most_common(top):
    print(f"{v:6d} {k}")
