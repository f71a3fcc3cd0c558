"""Summarise an `ncu --set full` capture of the fit kernels into profiles/ncu_summary.json.

usage: ncu_summary.py <report.ncu-rep> <out.json> "<source description>"

One entry per launch (kernel template argument SP: 1 = the standard space, 2 = the
disparity form, 3 = both); `dram_bytes_per_launch` (read + write) and, with a SASS source
page, `fp64_thread_inst_per_launch` (DFMA/DMUL/DADD/DSETP executed) are what bench.py reports
as `roofline.traffic` and `roofline.fp64`; "per_space" = the mean over the launches of a
two-launch step.

usage: ncu_summary.py <report.ncu-rep> <out.json> "<source description>"
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "dram__bytes.sum.per_second",
]
STALLS = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio")
NAMES = {"1": "standard", "2": "rgbd", "3": "both"}  # fit_tile_kernel<SP, ...>
UNIT_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def to_bytes(v: str) -> float:
    num, unit = v.split()
    return float(num) * UNIT_SCALE[unit]


def main() -> None:
    rep, out, source = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    summary = {"source": source, "dram_bytes_per_launch": {}, "kernels": {}}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        m = re.search(r"fit_tile_kernel<(\d)", name)
        if not m:
            continue
        form = NAMES[m.group(1)]
        k = {"kernel": name.split("(")[0]}
        for key in METRICS:
            if key in hdr:
                i = hdr.index(key)
                k[key] = f"{r[i]} {units[i]}".strip()
        stalls = {}
        for i, h in enumerate(hdr):
            s = STALLS.fullmatch(h)
            if s and not s.group(1).startswith("not_issued"):
                try:
                    stalls[s.group(1)] = round(float(r[i]), 3)
                except ValueError:
                    pass
        k["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:10])
        summary["kernels"][form] = k
        i_rd, i_wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        summary["dram_bytes_per_launch"][form] = (to_bytes(f"{r[i_rd]} {units[i_rd]}")
                                                  + to_bytes(f"{r[i_wr]} {units[i_wr]}"))
    # fp64 instructions per launch from the SASS source page (executed thread instructions)
    try:
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True, check=True).stdout
        fp64 = {}
        cur = None
        seen = set()
        for line in src.splitlines():
            if line.startswith('"Kernel Name"'):
                # the page lists each kernel's SASS twice: count the first copy
                m = re.search(r"fit_tile_kernel<\(int\)(\d)", line)
                cur = NAMES.get(m.group(1)) if m else None
                cur = None if cur in seen else cur
                if cur:
                    seen.add(cur)
                continue
            if cur is None or not line.startswith('"0x'):
                continue
            cols = next(csv.reader([line]))
            op = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9]+)", cols[1].strip())
            if op and op.group(2) in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
                fp64[cur] = fp64.get(cur, 0) + int(cols[6] or 0)  # thread instructions executed
        for form, n in fp64.items():
            summary["kernels"][form]["fp64_thread_inst_per_launch"] = n
    except Exception as e:  # noqa: BLE001
        summary["fp64_note"] = f"no SASS source page: {e}"
    ks = [summary["kernels"][k] for k in ("standard", "rgbd") if k in summary["kernels"]]
    if len(ks) == 2:
        def mean(key):
            try:
                return sum(float(str(k[key]).split()[0]) for k in ks) / 2
            except Exception:
                return None
        summary["kernels"]["per_space"] = {key: mean(key) for key in METRICS if mean(key) is not None}
        summary["kernels"]["per_space"]["fp64_thread_inst_per_launch"] = mean("fp64_thread_inst_per_launch")
        summary["dram_bytes_per_launch"]["per_space"] = (summary["dram_bytes_per_launch"]["standard"]
                                                         + summary["dram_bytes_per_launch"]["rgbd"]) / 2
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
        f.write("\n")
    print(json.dumps(summary["dram_bytes_per_launch"]))


if __name__ == "__main__":
    main()
