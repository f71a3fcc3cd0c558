"""Stall samples and executed instructions per source function region (by file:line -> the
enclosing function name found by scanning the source upward).
usage: stalls_by_fn.py <ncu source csv (sass)> <so> <kernel substring>"""
import collections, csv, glob, os, re, subprocess, sys, tempfile
src_csv, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, capture_output=True)
addr_loc = {}
for cubin in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
    cur, in_k = None, False
    for l in dis:
        if l.startswith("//----") and ".text." in l:
            in_k = kname in l; continue
        if not in_k: continue
        m = re.search(r'//## File "(.*)", line (\d+)', l)
        if m: cur = (m.group(1), int(m.group(2))); continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m and cur is not None: addr_loc[int(m.group(1), 16)] = cur
srcs = {}
def fn_of(path, line):
    if path not in srcs:
        try: srcs[path] = open(path).read().splitlines()
        except OSError: srcs[path] = []
    L = srcs[path]
    for i in range(min(line, len(L)) - 1, -1, -1):
        m = re.match(r'^(?:template <.*>\s*)?(?:__device__|__global__|static|inline|\w).*?\b(\w+)\s*\(', L[i])
        if L[i] and not L[i][0].isspace() and not L[i].startswith(("//", "#", "}")) and m:
            return os.path.basename(path) + ":" + m.group(1)
    return os.path.basename(path) + ":?"
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
isamp = hdr.index("Warp Stall Sampling (All Samples)")
base = min(int(r[ia], 16) for r in rows[2:] if len(r) > ia and r[ia].startswith("0x"))
inst = collections.Counter(); samp = collections.Counter(); st = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) <= ie or not r[ia].startswith("0x"): continue
    loc = addr_loc.get(int(r[ia], 16) - base)
    f = fn_of(*loc) if loc else "?"
    inst[f] += int(r[ie] or 0); samp[f] += int(r[isamp] or 0)
    for s in stalls: st[f][s] += int(r[hdr.index(s)] or 0)
ti, ts = sum(inst.values()), sum(samp.values())
for f, n in samp.most_common(25):
    top = ", ".join(f"{k[6:]} {v / max(1, n):.0%}" for k, v in st[f].most_common(4))
    print(f"{f:40s} inst {inst[f] / ti:6.1%}  samples {n / ts:6.1%}  [{top}]")
