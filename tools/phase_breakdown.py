"""Group ncu per-SASS samples by kernel phase (file + line ranges of the CUDA sources).
usage: phase_breakdown.py <ncu source csv (sass)> <so> <kernel mangled-name substring>"""
import collections, csv, glob, os, re, subprocess, sys, tempfile

src_csv, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, capture_output=True)
cubins = glob.glob(os.path.join(tmp, "*.cubin"))
addr_loc = {}
for cubin in cubins:
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
    cur, in_k = None, False
    for l in dis:
        if l.startswith("//----") and ".text." in l:
            in_k = kname in l
            continue
        if not in_k:
            continue
        m = re.search(r'//## File "(.*)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m and cur is not None:
            addr_loc[int(m.group(1), 16)] = cur
root = os.path.join(os.path.dirname(__file__), "..", "paper_2103_06644_b200", "csrc")
fit = open(os.path.join(root, "rf_fit.cu")).read().splitlines()


def line_of(marker):
    for i, l in enumerate(fit):
        if marker in l:
            return i + 1
    return 10 ** 9


marks = sorted([(line_of("__device__ __forceinline__ uint32_t smem_u32"), "tma_helpers"),
                (line_of("double primary_from_f32"), "primary"),
                (line_of("template <int VAR, bool USE_TMA, int RT, bool EXP>"), "kernel-setup"),
                (line_of("// ---- 1. halo tile -> primary"), "convert"),
                (line_of("// ---- 2. vertical window sums"), "vertical"),
                (line_of("// ---- 3/4. horizontal running sums"), "horizontal"),
                (line_of("      for (int j = 0; j < KSEG; ++j) {"), "pixel/C"),
                (line_of("          WindowFit f;"), "solve-call"),
                (line_of("      // ---- stores"), "stores")])


def phase(loc):
    if loc is None:
        return "?"
    f, ln = loc
    if f != "rf_fit.cu":
        return f
    p = "?"
    for s, n in marks:
        if ln >= s:
            p = n
    return p


rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = min(int(r[ia], 16) for r in rows[2:] if r[ia].startswith("0x"))
cnt, st = collections.Counter(), collections.Counter()
rs = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try:
        a = int(r[ia], 16) - base
        n = float(r[ie] or 0)
        s = float(r[iss] or 0)
    except Exception:
        continue
    ph = phase(addr_loc.get(a))
    cnt[ph] += n
    st[ph] += s
    for h in reasons:
        try:
            rs[ph][h] += float(r[hdr.index(h)] or 0)
        except Exception:
            pass
T, TS = sum(cnt.values()), sum(st.values())
print(f"total warp-instructions {T:.3e}")
for ph, n in sorted(cnt.items(), key=lambda x: -st[x[0]]):
    top = ", ".join(f"{k[6:]} {v / max(st[ph], 1) * 100:.0f}%" for k, v in rs[ph].most_common(4))
    print(f"{ph:14s} inst {n / T * 100:5.1f}%  stall-samples {st[ph] / TS * 100:5.1f}%  [{top}]")
