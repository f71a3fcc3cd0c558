"""Build the library plus experiment variants in parallel: build_variants.py name=FLAGS ...
(name 'main' = the in-tree librangefit_b200.so; others -> librangefit_b200_<name>.so)."""
import subprocess, sys
sys.path.insert(0, ".")
from paper_2103_06644_b200 import build as B

srcs = [str(s) for s in B.SOURCES]
base = [B.nvcc(), *B.NVCC_FLAGS, "-I", str(B.ROOT / "include")]
procs = {}
for arg in sys.argv[1:] or ["main="]:
    name, _, flags = arg.partition("=")
    out = B.OUT if name == "main" else B.PKG / f"librangefit_b200_{name}.so"
    procs[name] = subprocess.Popen(base + flags.split() + ["-o", str(out), *srcs], stdout=subprocess.PIPE,
                                   stderr=subprocess.PIPE, text=True)
rc = 0
for name, p in procs.items():
    o, e = p.communicate()
    if name == "main":
        (B.PKG / "ptxas_info.txt").write_text(e)
    errs = [l for l in e.splitlines() if "error" in l.lower()]
    print(name, "rc", p.returncode, *errs[:5])
    rc |= p.returncode
sys.exit(rc)
