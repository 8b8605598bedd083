"""Summarise an ncu --set full report (.ncu-rep) into the numbers the roofline
and DESIGN.md cite: duration, registers, occupancy, FP64 pipe, issue, DRAM
bytes / throughput, local-memory traffic, top stall reasons and the SASS
opcode mix weighted by executed instructions.

usage: python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...]
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("duration_us", "gpu__time_duration.sum", 1e-3),
    ("registers", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
    ("achieved_occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("fp64_pipe_pct_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("threads_per_warp_inst", "smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    ("warp_inst_executed", "smsp__inst_executed.sum", 1),
    ("dram_read_bytes", "dram__bytes_read.sum", 1),
    ("dram_write_bytes", "dram__bytes_write.sum", 1),
    ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("local_load_inst", "sass__inst_executed_local_loads", 1),
    ("local_store_inst", "sass__inst_executed_local_stores", 1),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6, "nsecond": 1, "ns": 1, "us": 1e3}


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout


def summarise(path):
    out = []
    raw = list(csv.reader(io.StringIO(ncu(["-i", path, "--page", "raw", "--csv"]))))
    head, units = raw[0], raw[1]
    for row in raw[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        out.append(f"== {d.get('Kernel Name', '?')[:110]}")
        for name, key, _ in KEYS:
            if key not in d:
                continue
            v = d[key].replace(",", "")
            try:
                if key == "gpu__time_duration.sum":
                    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
                    x = float(v) * scale.get(u.get(key, ""), 1.0)  # -> us
                else:
                    x = float(v) * UNIT_SCALE.get(u.get(key, ""), 1)
                v = f"{x:.6g}"
            except ValueError:
                pass
            out.append(f"  {name:28s} {v}")
        st = {}
        for k, v in d.items():
            mt = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
            if mt and v:
                st[mt.group(1)] = float(v)
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        out.append("  stalls (warps per issue): " + ", ".join(f"{k} {v:.2f}" for k, v in top))
    # opcode mix (first kernel in the report)
    src = list(csv.reader(io.StringIO(ncu(["-i", path, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        h = src[1]
        iS, iE = h.index("Source"), h.index("Instructions Executed")
        ops = collections.Counter()
        for r in src[2:]:
            try:
                e = int(r[iE] or 0)
            except (ValueError, IndexError):
                continue
            txt = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
            op = "IMAD.MOV" if txt.startswith("IMAD.MOV") else txt.split(" ")[0].split(".")[0]
            ops[op] += e
        tot = sum(ops.values()) or 1
        out.append("  SASS mix (executed): " + ", ".join(f"{o} {c / tot * 100:.1f}%" for o, c in ops.most_common(12)))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"# {p}")
        print(summarise(p))
