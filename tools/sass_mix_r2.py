"""Static SASS opcode mix of the per-pixel tile kernels (cuobjdump of the in-tree library) and,
from an ncu --set full report, the executed mix per pixel-fit: the Blackwell-native evidence
(UTMALDG = TMA tensor loads, SYNCS = mbarrier, FFMA2/FMUL2/FADD2 = packed fp32 pairs, DFMA...).
usage: sass_mix_r2.py <report.ncu-rep> <pixel-fits per launch> > profiles/sass_mix_r2.txt"""
import collections, csv, re, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SO = ROOT / "paper_2103_06644_b200" / "librangefit_b200.so"
KEYS = ["UTMALDG", "SYNCS", "BAR", "DFMA", "DMUL", "DADD", "DSETP", "FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL",
        "MUFU", "F2F", "LDS", "STS", "LDG", "STG", "SHFL", "REDUX", "ATOMS"]
sass = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True, check=True).stdout
static = collections.defaultdict(collections.Counter)
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9]+)", line)
    if cur and m:
        static[cur][m.group(2)] += 1
print("# Static SASS of fit_tile_kernel<SP, TMA, RT, EXP> (SP 1 standard, 2 disparity form, 3 both;")
print("# RT = compile-time window radius), counts per kernel body: " + ", ".join(KEYS))
for name in sorted(static):
    m = re.search(r"fit_tile_kernelILi(\d)ELb(\d)ELi(\d+)ELb(\d)E", name)
    if not m or m.group(2) != "1" or m.group(3) not in ("2", "4", "7", "15") or m.group(4) != "0":
        continue
    c = static[name]
    print(f"fit_tile_kernel<SP={m.group(1)}, TMA, r={m.group(3)}>  total {sum(c.values())}  " +
          " ".join(f"{k}={c[k]}" for k in KEYS))
if len(sys.argv) > 2:
    rep, pix = sys.argv[1], float(sys.argv[2])
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    execd = collections.defaultdict(collections.Counter)
    cur, seen = None, set()
    for line in src.splitlines():
        if line.startswith('"Kernel Name"'):
            m = re.search(r"fit_tile_kernel<\(int\)(\d), \(bool\)1, \(int\)(\d+)", line)
            cur = f"SP={m.group(1)}, r={m.group(2)}" if m else None
            cur = None if cur in seen else cur
            if cur:
                seen.add(cur)
            continue
        if cur is None or not line.startswith('"0x'):
            continue
        cols = next(csv.reader([line]))
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9]+)", cols[1].strip())
        if m:
            execd[cur][m.group(2)] += int(cols[5] or 0) * 32  # warp instructions x 32
    print(f"\n# Executed (ncu --set full {Path(rep).name}): thread instructions per pixel-fit "
          f"({pix:.0f} pixel-fits per launch)")
    for k, c in execd.items():
        tot = sum(c.values())
        fp64 = sum(c[o] for o in ("DFMA", "DMUL", "DADD", "DSETP"))
        xu = sum(c[o] for o in ("MUFU", "F2F", "I2F", "F2I"))
        print(f"fit_tile_kernel<{k}>  all {tot / pix:.1f}  fp64 {fp64 / pix:.1f}  xu {xu / pix:.1f}  " +
              " ".join(f"{o}={c[o] / pix:.2f}" for o in KEYS if c[o]))
