"""Executed-instruction opcode mix per kernel phase (same phases as phase_breakdown.py).
usage: phase_ops.py <ncu source csv (sass)> <so> <kernel substring>"""
import collections, csv, sys, runpy
sys.argv = sys.argv[:4]
ns = runpy.run_path(__file__.replace("phase_ops.py", "phase_breakdown.py"), run_name="pb")
phase, addr_loc = ns["phase"], ns["addr_loc"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
base = min(int(r[ia], 16) for r in rows[2:] if r[ia].startswith("0x"))
ops = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try:
        a = int(r[ia], 16) - base
        n = float(r[ie] or 0)
    except Exception:
        continue
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    loc = addr_loc.get(a)
    ph = phase(loc)
    if ph == "rf_solve.cuh":
        ph = "solve:%d" % (loc[1] // 20 * 20)
    ops[ph][op.split(".")[0]] += n
T = sum(sum(c.values()) for c in ops.values())
print("\n=== per phase")
for ph, c in sorted(ops.items(), key=lambda x: -sum(x[1].values())):
    tot = sum(c.values())
    print(f"{ph:16s} {tot / T * 100:5.1f}%  " + ", ".join(f"{k} {v / tot * 100:.0f}" for k, v in c.most_common(8)))
