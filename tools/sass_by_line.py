"""Aggregate ncu per-SASS metrics by CUDA source line.
usage: sass_by_line.py <ncu source csv (sass)> <so file> <kernel substring> [topN]"""
import collections, csv, re, subprocess, sys, tempfile, os, glob

src_csv, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
addr_line = {}
cur_line = None
in_k = False
for l in dis:
    if l.startswith("//----") and ".text." in l:
        in_k = kname in l
        continue
    if not in_k:
        continue
    m = re.search(r'//## File ".*", line (\d+)', l)
    if m:
        cur_line = int(m.group(1))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and cur_line is not None:
        addr_line[int(m.group(1), 16)] = cur_line
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia = hdr.index("Address"); ie = hdr.index("Instructions Executed"); iss = hdr.index("Warp Stall Sampling (All Samples)")
cnt = collections.Counter(); st = collections.Counter()
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
        base = a if base is None else min(base, a)
    except Exception:
        pass
for r in rows[2:]:
    try:
        a = int(r[ia], 16); n = float(r[ie] or 0); s = float(r[iss] or 0)
    except Exception:
        continue
    ln = addr_line.get(a - base, -1)
    cnt[ln] += n; st[ln] += s
tot = sum(cnt.values()); tots = sum(st.values())
srcl = open(os.path.join(os.path.dirname(__file__), "..", "paper_2103_06644_b200", "csrc", "rf_fit.cu")).read().splitlines()
for ln, n in cnt.most_common(top):
    text = srcl[ln - 1].strip()[:90] if 0 < ln <= len(srcl) else "?"
    print(f"L{ln:4d} {n/tot*100:5.1f}% inst {st[ln]/tots*100:5.1f}% stall | {text}")
