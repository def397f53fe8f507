"""Compact per-launch summary of an ncu --set full report (.ncu-rep):
duration, DRAM bytes, DRAM/SM throughput, IPC, occupancy, registers, pipe
utilisation and the top warp-stall reasons - plus (--traffic out.json) the
per-kernel DRAM traffic per launch that bench.py reports as roofline.traffic.

  python profiles/ncu_summary.py gpurun_out/prof/full_f12.ncu-rep [--traffic profiles/traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "dur_us", 1e-3),
    ("dram__bytes_read.sum", "dram_rd_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_wr_MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1),
    ("sm__inst_executed.avg.per_cycle_active", "ipc", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_%", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_%", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_%", 1),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%", 1),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    path = sys.argv[1]
    traffic_out = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    rows, units = raw(path)
    cols = ["kernel"] + [m[1] for m in METRICS] + ["top stalls"]
    print(" | ".join(cols))
    traffic = {}
    for r in rows:
        name = r.get("Kernel Name", "?").split("(")[0].replace("vms::<unnamed>::", "")
        name = name.replace("unnamed>::", "").replace("void ", "")
        vals = []
        for key, label, scale in METRICS:
            v = num(r.get(key, "nan"))
            u = units.get(key, "")
            if key.startswith("gpu__time"):  # -> ns, then the 1e-3 scale -> us
                v *= {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                      "msecond": 1e6, "s": 1e9, "second": 1e9}.get(u, 1.0)
            if key.startswith("dram__bytes"):  # -> bytes
                v *= {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u.lower(), 1.0)
            vals.append(v * scale)
        stalls = sorted(((num(v), k) for k, v in r.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                        reverse=True)[:3]
        st = ", ".join(k.replace("smsp__pcsamp_warps_issue_stalled_", "") for _, k in stalls if _ == _)
        print(" | ".join([name] + [f"{v:.3g}" for v in vals] + [st]))
        base = name.split("<")[0]
        rd, wr = vals[1], vals[2]
        m = dict(zip([x[1] for x in METRICS], vals))
        traffic.setdefault(base, []).append(
            ((rd + wr) * 1e6, m["dur_us"], m["fp64_%"], m["xu_%"], m["ipc"], m["sm_%"], st))
    if traffic_out:
        def mean(v, i):
            return round(sum(x[i] for x in v) / len(v), 3)

        frame = next((tok[1:] for tok in path.replace(".", "_").split("_")
                      if tok.startswith("f") and tok[1:].isdigit()), None)
        summary = {k: {"bytes_per_launch": mean(v, 0), "launches": len(v), "dur_us": mean(v, 1),
                       "fp64_pct": mean(v, 2), "xu_pct": mean(v, 3), "ipc": mean(v, 4),
                       "issue_frac": round(mean(v, 4) / 4.0, 3), "sm_pct": mean(v, 5),
                       "top_stalls": v[0][6], "frame": frame,
                       "source": path.split("/")[-1]} for k, v in traffic.items()}
        with open(traffic_out, "w") as fh:
            json.dump(summary, fh, indent=1)
        print("traffic ->", traffic_out)


if __name__ == "__main__":
    main()
