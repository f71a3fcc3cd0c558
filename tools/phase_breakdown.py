"""Group ncu per-SASS samples by kernel phase using line ranges of rf_fit.cu."""
import collections, csv, re, subprocess, sys, tempfile, os, glob
src_csv, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
addr_line, cur, in_k = {}, None, False
for l in dis:
    if l.startswith("//----") and ".text." in l:
        in_k = kname in l; continue
    if not in_k: continue
    m = re.search(r'//## File ".*", line (\d+)', l)
    if m: cur = int(m.group(1)); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and cur is not None: addr_line[int(m.group(1), 16)] = cur
src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2103_06644_b200", "csrc", "rf_fit.cu")).read().splitlines()
# phase markers: first line index containing each marker
marks = [("helpers", "// ------------------------------------------------------------------ helpers"),
         ("tma_helpers", "// residue-major column stride"),
         ("convert", "    // ---- 1. halo tile -> primary"),
         ("solve", "__device__ __forceinline__ void solve_window"),
         ("finish", "__device__ __forceinline__ void finish_plane"),
         ("primary", "// depth element -> fp64 primary p"),
         ("kernel-setup", "template <int VAR, bool USE_TMA>"),
         ("vertical", "    // ---- 2. vertical running sums"),
         ("horizontal", "    // ---- 3/4. horizontal running sums"),
         ("pixel/C", "      for (int j = 0; j < KSEG; ++j) {"),
         ("tables", "// ------------------------------------------------------------------ tables")]
starts = []
for name, m in marks:
    first = m.split("\n")[0]
    for i, l in enumerate(src):
        if l.startswith(first) or l.strip() == first.strip():
            starts.append((i + 1, name)); break
starts.sort()
def phase(line):
    p = "?"
    for s, n in starts:
        if line >= s: p = n
    return p
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = min(int(r[ia], 16) for r in rows[2:] if r[ia].startswith("0x"))
cnt, st = collections.Counter(), collections.Counter()
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
rs = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try: a = int(r[ia], 16) - base; n = float(r[ie] or 0); s = float(r[iss] or 0)
    except Exception: continue
    ph = phase(addr_line.get(a, -1))
    cnt[ph] += n; st[ph] += s
    for h in reasons:
        try: rs[ph][h] += float(r[hdr.index(h)] or 0)
        except Exception: pass
T, TS = sum(cnt.values()), sum(st.values())
for ph, n in sorted(cnt.items(), key=lambda x: -st[x[0]]):
    top = ", ".join(f"{k[6:]} {v/max(st[ph],1)*100:.0f}%" for k, v in rs[ph].most_common(4))
    print(f"{ph:12s} inst {n/T*100:5.1f}%  stall-samples {st[ph]/TS*100:5.1f}%  [{top}]")
