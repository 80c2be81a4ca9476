"""Summarise an ncu report (or a launch-list CSV) into profiles/ (tracked).

    python tools/ncu_summary.py gpurun_out/prof_scan.ncu-rep profiles/r01_scan_N64.md
    python tools/ncu_summary.py gpurun_out/launches.csv profiles/r01_launches.md
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
        "sm__cycles_elapsed.avg", "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_utcmma.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def from_rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "")[:90]}
        for k in KEYS:
            if k in d:
                ent[k] = f"{d[k]} {u.get(k, '')}".strip()
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and d[k] not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        ent["top_stalls"] = ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:5])
        out.append(ent)
    return out


def from_csv(path):
    rows = list(csv.reader(open(path)))
    i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    agg = {}
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", ""))
    return agg


def main(src, dst):
    with open(dst, "w") as f:
        if src.endswith(".csv"):
            agg = from_csv(src)
            tot = sum(v[1] for v in agg.values()) or 1.0
            f.write(f"# ncu launch list: {src}\n\n(cold-cache, serialised: compare SHARES, not absolutes)\n\n")
            f.write("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
            for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
                f.write(f"| {k} | {n} | {ns / 1e3:.1f} | {ns / n / 1e3:.2f} | {ns / tot:.1%} |\n")
        else:
            f.write(f"# ncu --set full summary: {src}\n\n")
            for e in from_rep(src):
                f.write(f"## {e.pop('kernel')}\n\n")
                for k, v in e.items():
                    f.write(f"- {k}: {v}\n")
                f.write("\n")
    print(open(dst).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
