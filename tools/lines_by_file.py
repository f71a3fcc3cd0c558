"""Top source lines (file:line) by executed instructions for one kernel.
usage: lines_by_file.py <ncu source csv> <so> <kernel substring> [file filter] [topN]"""
import collections, csv, glob, os, re, subprocess, sys, tempfile
src_csv, so, kname = sys.argv[1:4]
ffilter = sys.argv[4] if len(sys.argv) > 4 else ""
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
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
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
base = min(int(r[ia], 16) for r in rows[2:] if r[ia].startswith("0x"))
cnt = collections.Counter()
for r in rows[2:]:
    try: a = int(r[ia], 16) - base; n = float(r[ie] or 0)
    except Exception: continue
    cnt[addr_loc.get(a, ("?", 0))] += n
T = sum(cnt.values())
cache = {}
for (f, ln), n in cnt.most_common():
    if ffilter and ffilter not in f: continue
    if f not in cache:
        try: cache[f] = open(f).read().splitlines()
        except Exception: cache[f] = []
    txt = cache[f][ln - 1].strip()[:95] if 0 < ln <= len(cache[f]) else ""
    print(f"{os.path.basename(f)}:{ln:<4d} {n/T*100:5.2f}% | {txt}")
    top -= 1
    if top <= 0: break
