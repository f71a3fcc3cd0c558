"""Print the SASS of one kernel for a source-line range of rf_fit.cu / rf_solve.cuh.
usage: sass_lines.py <so> <kernel substring> <file basename> <line0> <line1>"""
import glob, os, re, subprocess, sys, tempfile
so, kname, fname, l0, l1 = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, capture_output=True)
for cubin in glob.glob(os.path.join(tmp, "*.cubin")):
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
        if cur and cur[0] == fname and l0 <= cur[1] <= l1 and re.match(r'\s*/\*[0-9a-f]{4,}\*/', l):
            print(f"{cur[1]:4d} {l.strip()[:110]}")
