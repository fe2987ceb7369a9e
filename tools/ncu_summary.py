"""Summarise ncu output for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.txt
    python tools/ncu_summary.py report gpurun_out/x.ncu-rep [...]  > profiles/rNN_ncu_full.json
    python tools/ncu_summary.py traffic "<source>" chacha20=gpurun_out/c20.ncu-rep [...] > profiles/ncu_traffic.json
"""

import collections
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_math_pipe_throttle",
]
STALL_RE = re.compile(r"smsp__pcsamp_warps_issue_stalled_(\w+)$")


def launches(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki])[:70]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# ncu launch list summary of {path}: {sum(cnt.values())} launches, {T / 1e3:.1f} us total device time")
    print("# (cold-cache, serialised by ncu: compare shares, not absolutes)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / 1e3:12.1f} us {100 * v / T:6.2f}%  n={cnt[k]:6d}  avg={v / cnt[k] / 1e3:9.2f} us  {k}")


def report(paths):
    out = {}
    for p in paths:
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(h, r))
            key = f"{p.split('/')[-1]}::{re.sub(r'[(<].*', '', d.get('Kernel Name', ''))}#{d.get('ID')}"
            m = {}
            for name in METRICS:
                if name in d and d[name] not in ("", "n/a"):
                    u = units[h.index(name)]
                    m[name] = f"{d[name]} {u}".strip()
            stalls = {}
            for i, name in enumerate(h):
                mm = STALL_RE.match(name)
                if mm and r[i] not in ("", "n/a"):
                    try:
                        stalls[mm.group(1)] = float(r[i].replace(",", ""))
                    except ValueError:
                        pass
            tot = sum(stalls.values()) or 1.0
            m["stall_samples_top"] = {k: round(100 * v / tot, 1) for k, v in
                                      sorted(stalls.items(), key=lambda x: -x[1])[:6]}
            m["kernel_full_name"] = d.get("Kernel Name", "")
            out[key] = m
    print(json.dumps(out, indent=1))


def _num(v):
    return float(str(v).split()[0].replace(",", ""))


def traffic(source, specs):
    """profiles/ncu_traffic.json from one --set full report per bench kernel:
    specs = name=path.ncu-rep[:pages] (name as bench.py looks it up:
    chacha20, chacha12_desc, ...)."""
    out = {"source": source}
    for spec in specs:
        name, path = spec.split("=", 1)
        pages = 262144
        if ":" in path:
            path, pg = path.rsplit(":", 1)
            pages = int(pg)
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        d = dict(zip(h, rows[2]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = _num(d["dram__bytes_read.sum"]) * scale[units[h.index("dram__bytes_read.sum")]]
        wr = _num(d["dram__bytes_write.sum"]) * scale[units[h.index("dram__bytes_write.sum")]]
        dur = _num(d["gpu__time_duration.sum"]) * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(
            units[h.index("gpu__time_duration.sum")], 1)
        stalls = {}
        for i, col in enumerate(h):
            mm = STALL_RE.match(col)
            if mm and rows[2][i] not in ("", "n/a"):
                stalls[mm.group(1)] = _num(rows[2][i])
        tot = sum(stalls.values()) or 1.0
        out[name] = {
            "kernel": re.sub(r"\(.*", "", d.get("Kernel Name", "")), "pages": pages,
            "dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
            "algorithmic_bytes": pages * 8192 + (12 * pages if name.endswith("_desc") else 0),
            "duration_us": round(dur, 3),
            "alu_pipe_pct": d.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "dram_throughput_pct": d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "registers": d.get("launch__registers_per_thread"), "grid": d.get("launch__grid_size"),
            "sm_clock_ghz": d.get("sm__cycles_elapsed.avg.per_second"),
            "stalls": {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]},
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    else:
        report(sys.argv[2:])
