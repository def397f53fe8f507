"""Summarise VMSPLAT_TRACE=2 per-frame timelines ([tl] lines on stderr).

Per frame: host waits (visibility, recycle), device visibility, front and
blend durations, the gap between consecutive blends on the caller's stream,
and the spacing of the image copies (host output).  Usage:
    python scripts/tl_summary.py LOG [--frames]
"""
import sys


def rows(path):
    out = []
    for line in open(path):
        if not line.startswith("[tl]"):
            continue
        t = line.split()
        v = [float(x) for x in (t[3], t[4], t[5], t[6], t[9], t[10], t[12], t[13], t[16])]
        ext = [float(t[19]), float(t[22])] if len(t) > 22 else [0.0, 0.0]
        out.append(v + ext)
    return out


def main():
    path = sys.argv[1]
    r = rows(path)[-32:]
    keys = ("vis_wait", "recycle", "vis", "front", "blend", "blend_gap", "d2h_step")
    acc = {k: [] for k in keys}
    prev_be = prev_d2h = None
    for (he, hv, hq, hx, vs, ve, rs, re, d2h, fe, bs) in r:
        row = {"vis_wait": hv - he, "recycle": hq - hv, "vis": ve - vs, "front": fe - rs,
               "blend": re - bs}
        row["blend_gap"] = bs - prev_be if prev_be is not None else None
        row["d2h_step"] = d2h - prev_d2h if (prev_d2h is not None and d2h > 0) else None
        prev_be, prev_d2h = re, d2h
        for k in keys:
            if row[k] is not None:
                acc[k].append(row[k])
        if "--frames" in sys.argv:
            print(" ".join(f"{k} {row[k]:7.0f}" if row[k] is not None else f"{k}       -"
                           for k in keys))
    print("mean (us):", ", ".join(f"{k} {sum(v) / len(v):.0f}" for k, v in acc.items() if v))


if __name__ == "__main__":
    main()
