"""Per-source-line warp-stall samples of one kernel in an ncu report (--set full with
--import-source on, -lineinfo build): the lines where the kernel's time goes.

    python tools/ncu_lines.py gpurun_out/prof_tail_N48.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    fname, hdr, out = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            d = dict(zip(hdr[2:], r[2:]))
            d["Source"] = r[1]
            s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
            if s > 0:
                out.append((s, fname, int(r[0]), d.get("Source", "").strip()[:100]))
    tot = sum(x[0] for x in out) or 1
    for s, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{s / tot:6.1%} {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
