#!/usr/bin/env python
"""Equal-resolution comparison of TGV diagnostic histories (tools/tgv_history.py output), as the
paper's high-speed TGV study (Table TGV-sup-4): deviations of E_k(t) and eps_S(t) of each
run from a reference run (linear interpolation in t), the device time each run spent stepping, and
an SVG figure of both histories (no plotting library needed).

  python tools/tgv_compare.py REF.jsonl RUN1.jsonl [RUN2.jsonl ...] [--svg out.svg]
"""
import json
import sys

import numpy as np


def load(path):
    rows, meta = [], None
    for line in open(path):
        d = json.loads(line)
        if "E_k" in d:
            rows.append((d["t"], d["E_k"], d["eps_S"], d["eps_D"], d["eps_T"]))
        else:
            meta = d
    return np.array(rows), meta


def label(meta):
    return f"{meta['scheme'].upper().replace('CGKS5', 'CGKS-5th').replace('GKS2', 'GKS-2nd')} {meta['n']}^3"


def svg(series, path, t_max):
    W, H, pad = 900, 380, 50
    pw = (W - 3 * pad) / 2
    colors = ["#000000", "#d62728", "#1f77b4", "#2ca02c"]
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" font-family="sans-serif" font-size="12">',
           f'<rect width="{W}" height="{H}" fill="white"/>']
    for p, (col, name) in enumerate([(1, "E_k"), (2, "eps_S")]):
        x0 = pad + p * (pw + pad)
        ymax = max(s[0][:, col].max() for s in series) * 1.05
        out.append(f'<rect x="{x0}" y="{pad}" width="{pw}" height="{H - 2 * pad}" fill="none" stroke="#888"/>')
        out.append(f'<text x="{x0 + pw / 2}" y="{pad - 10}" text-anchor="middle">{name}(t)</text>')
        for k in range(6):
            tv = t_max * k / 5
            X = x0 + pw * k / 5
            out.append(f'<text x="{X}" y="{H - pad + 15}" text-anchor="middle">{tv:.0f}</text>')
            yv = ymax * k / 5
            Y = H - pad - (H - 2 * pad) * k / 5
            out.append(f'<text x="{x0 - 5}" y="{Y + 4}" text-anchor="end">{yv:.3g}</text>')
        for si, (arr, meta) in enumerate(series):
            pts = " ".join(f"{x0 + pw * t / t_max:.1f},{H - pad - (H - 2 * pad) * v / ymax:.1f}"
                           for t, v in zip(arr[:, 0], arr[:, col]) if t <= t_max)
            out.append(f'<polyline fill="none" stroke="{colors[si % 4]}" stroke-width="1.5" points="{pts}"/>')
            if p == 0:
                out.append(f'<text x="{x0 + pw - 5}" y="{pad + 18 + 16 * si}" text-anchor="end" '
                           f'fill="{colors[si % 4]}">{label(meta)}</text>')
    out.append("</svg>")
    open(path, "w").write("\n".join(out))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out_svg = None
    if "--svg" in sys.argv:
        out_svg = sys.argv[sys.argv.index("--svg") + 1]
        args.remove(out_svg)
    ref, rmeta = load(args[0])
    series = [(ref, rmeta)]
    res = {"reference": {"run": label(rmeta), "device_seconds": rmeta["device_seconds_stepping"],
                         "steps": rmeta["steps"]}, "runs": []}
    for p in args[1:]:
        arr, meta = load(p)
        series.append((arr, meta))
        t = arr[:, 0]
        m = t <= ref[-1, 0]
        row = {"run": label(meta), "device_seconds": meta["device_seconds_stepping"], "steps": meta["steps"]}
        for col, name in [(1, "E_k"), (2, "eps_S"), (4, "eps_T")]:
            r = np.interp(t[m], ref[:, 0], ref[:, col])
            d = arr[m, col] - r
            row[f"{name}_max_abs_dev_rel"] = float(np.abs(d).max() / np.abs(ref[:, col]).max())
            row[f"{name}_rms_dev_rel"] = float(np.sqrt((d ** 2).mean()) / np.abs(ref[:, col]).max())
        res["runs"].append(row)
    base = res["runs"][0]["device_seconds"] if res["runs"] else None
    for row in res["runs"]:
        row["time_ratio_to_first_run"] = row["device_seconds"] / base
    print(json.dumps(res, indent=1))
    if out_svg:
        svg(series, out_svg, float(min(s[0][-1, 0] for s in series)))


if __name__ == "__main__":
    main()
