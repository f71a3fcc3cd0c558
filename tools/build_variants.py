"""Build the library plus experiment variants: build_variants.py name=FLAGS ...
(name 'main' = the in-tree librangefit_b200.so; others -> librangefit_b200_<name>.so)."""
import sys
sys.path.insert(0, ".")
from paper_2103_06644_b200 import build as B

rc = 0
for arg in sys.argv[1:] or ["main="]:
    name, _, flags = arg.partition("=")
    out = B.OUT if name == "main" else B.PKG / f"librangefit_b200_{name}.so"
    try:
        B.build(force=True, out=out, extra_flags=flags.split())
        print(name, "rc 0")
    except RuntimeError as e:
        print(name, "rc 1", str(e)[-2000:])
        rc = 1
sys.exit(rc)
