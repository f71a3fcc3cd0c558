"""Executed-instruction opcode mix per source file (thread instr per pixel-fit).
usage: opmix.py <ncu source csv (sass)> <so> <kernel substring> <pixel-fits> [file]"""
import collections, csv, glob, os, re, subprocess, sys, tempfile
src_csv, so, kname, pix = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
ffilter = sys.argv[5] if len(sys.argv) > 5 else None
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
        if m: cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m and cur is not None: addr_loc[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
base = min(int(r[ia], 16) for r in rows[2:] if len(r) > ia and r[ia].startswith("0x"))
ops = collections.Counter(); byfile = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie or not r[ia].startswith("0x") or not r[ie].isdigit(): continue
    loc = addr_loc.get(int(r[ia], 16) - base, ("?", 0))
    n = int(r[ie]) * 32 / pix
    byfile[loc[0]] += n
    if ffilter and loc[0] != ffilter: continue
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9]+)(\.[A-Z0-9_.]+)?', r[isrc].strip())
    if m: ops[m.group(2)] += n
print({k: round(v, 1) for k, v in byfile.most_common()})
print("total", round(sum(ops.values()), 1))
for k, v in ops.most_common(40): print(f"  {k:12s} {v:7.1f}")
