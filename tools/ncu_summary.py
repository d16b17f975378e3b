"""Summarise an ncu --set full report: duration, DRAM/L2/shared traffic,
instruction mix and stall reasons of the profiled kernel (JSON to stdout).

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [--sass]
"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

NCU = "/usr/local/cuda/bin/ncu"


def page(rep, name, extra=()):
    out = subprocess.run([NCU, "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = page(rep, "raw")
    if len(rows) > 3:  # several profiled launches (e.g. a two-class split): raw metrics of each
        outs = [summarise(rows[0], rows[1], r) for r in rows[2:]]
        tot = {k: sum(o[k] or 0 for o in outs) for k in ("duration_s", "dram_read_bytes", "dram_write_bytes",
                                                          "l2_read_bytes_from_sm", "smem_wavefronts", "inst_executed")}
        print(json.dumps({"launches": outs, "sum": tot}, indent=1))
        return
    out = summarise(rows[0], rows[1], rows[2])
    src = page(rep, "source", ["--print-source", "sass"])
    h = src[1]
    data = src[2:]
    scols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in scols}
    T = sum(tot.values()) or 1
    out["stalls_pct"] = {c[6:]: round(v / T * 100, 1) for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v / T > 0.005}
    iE = h.index("Instructions Executed")
    mix = Counter()
    for r in data:
        t = r[1].split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        mix[op] += float(r[iE] or 0)
    out["inst_mix_M"] = {k: round(v / 1e6, 1) for k, v in mix.most_common(14)}
    print(json.dumps(out, indent=1))


def summarise(hdr, units, vals):
    raw = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}

    def num(k):
        v, u = raw.get(k, ("nan", ""))
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            return None
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                 "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
        return x * scale

    dur = num("gpu__time_duration.sum")
    out = {
        "kernel": raw.get("Kernel Name", ("?",))[0][:120],
        "duration_s": dur,
        "dram_read_bytes": num("dram__bytes_read.sum"),
        "dram_write_bytes": num("dram__bytes_write.sum"),
        "l2_bytes": num("lts__t_bytes.sum"),
        "l2_read_bytes_from_sm": num("lts__t_sectors_srcunit_tex_op_read.sum") and num("lts__t_sectors_srcunit_tex_op_read.sum") * 32,
        "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_wavefront_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "inst_executed": num("sm__inst_executed.sum"),
        "issue_pct": num("sm__inst_executed.sum.pct_of_peak_sustained_elapsed"),
        "sm_clock_hz": num("sm__cycles_elapsed.avg.per_second"),
        "registers": num("launch__registers_per_thread"),
    }
    return out


if __name__ == "__main__":
    main()
