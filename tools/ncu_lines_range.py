"""Per-source-line warp-stall samples (all launches of an ncu report aggregated), with the
top stall reasons, optionally restricted to line ranges of one file (diagnostics).

    python tools/ncu_lines_range.py REP k_tail.cu 129-340,713-822
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, fname_want, ranges):
    rg = [tuple(int(v) for v in x.split("-")) for x in ranges.split(",")] if ranges else []
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = hdr = None
    agg = defaultdict(lambda: [0.0, defaultdict(float), ""])
    for r in csv.reader(io.StringIO(raw)):
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not (hdr and len(r) == len(hdr) and r[0].isdigit()) or fname != fname_want:
            continue
        ln = int(r[0])
        if rg and not any(a <= ln <= b for a, b in rg):
            continue
        d = dict(zip(hdr[2:], r[2:]))
        s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        if s <= 0:
            continue
        e = agg[ln]
        e[0] += s
        e[2] = r[1].strip()[:64]
        for h in hdr[2:]:
            if h.startswith("stall_") and "Not Issued" not in h:
                e[1][h[6:]] += float(d[h] or 0)
    tot = sum(e[0] for e in agg.values())
    print(f"total samples {tot:.0f}")
    for ln in sorted(agg):
        s, st, src = agg[ln]
        top = sorted(((v, k) for k, v in st.items() if v > 0), reverse=True)[:3]
        print(f"{ln:5d} {s:7.0f} {src:64s} " + " ".join(f"{k}:{v:.0f}" for v, k in top))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
