"""Mutation check of the oracle's pins (CPU, diagnostics).

    python tools/oracle_mutants.py [--only SUBSTR]

Applies one plausible slip at a time to oracle/argus_oracle.c or oracle/control.py
(a dropped term, a flipped comparison, a wrong index or sign), rebuilds, and runs
the oracle pin tests (tests/test_oracle_*.py, -x).  A mutant that passes every pin
"survives": the pins cannot tell it from the paper's definition.  The sources are
restored after every mutant (and on interruption).  Prints one line per mutant and
a JSON summary.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C = "oracle/argus_oracle.c"
PY = "oracle/control.py"

MUTANTS = [
    # O1 bf16 rounding
    ("bf16 ties away from zero", C, "if (lower > 0x8000u || (lower == 0x8000u && (upper & 1u))) upper += 1u;",
     "if (lower >= 0x8000u) upper += 1u;"),
    ("bf16 ties to odd", C, "(lower == 0x8000u && (upper & 1u))", "(lower == 0x8000u && !(upper & 1u))"),
    ("bf16 truncation", C, "if (lower > 0x8000u || (lower == 0x8000u && (upper & 1u))) upper += 1u;", ""),
    # O2/O3 cosine
    ("cosine without the cache norm", C, "double s = dot / (nx * nc[j]);", "double s = dot / nx;"),
    ("cosine squared norm", C, "nc[j] = sqrt(q);", "nc[j] = q;"),
    ("cosine fp32 input (no bf16 of X)", C, "for (int64_t e = 0; e < (int64_t)N * d; ++e) Xb[e] = (float)orc_bf16(X[e]);",
     "for (int64_t e = 0; e < (int64_t)N * d; ++e) Xb[e] = X[e];"),
    ("pair cosine without the x norm", C, "return dot_bf16(x, c, d) / (nx * nc);", "return dot_bf16(x, c, d) / nc;"),
    # O4 top-k
    ("ties to the newer entry", C, "return s > s2 || (s == s2 && g < g2);", "return s > s2 || (s == s2 && g > g2);"),
    ("top-k ascending", C, "return s > s2 || (s == s2 && g < g2);", "return s < s2 || (s == s2 && g < g2);"),
    ("padding score 0", C, "for (int32_t t = 0; t < k; ++t) { bs[t] = -1.0; bg[t] = 0xFFFFFFFFu; }\n        if (!(nx",
     "for (int32_t t = 0; t < k; ++t) { bs[t] = 0.0; bg[t] = 0xFFFFFFFFu; }\n        if (!(nx"),
    ("ids ignored", C, "uint32_t g = ids ? ids[j] : (uint32_t)j;", "uint32_t g = (uint32_t)j;"),
    # O5 predictor
    ("no ReLU", C, "h[j] = a > 0.0 ? a : 0.0;", "h[j] = a;"),
    ("no b1", C, "a += (double)b1[j];", ""),
    ("no b2", C, "double z = (double)b2[v];", "double z = 0.0;"),
    ("r_0 not pinned to 1", C, "rhat[(int64_t)i * L + 0] = 1.0; /*", "/*"),
    ("sigmoid sign", C, "1.0 / (1.0 + exp(-z))", "1.0 / (1.0 + exp(z))"),
    ("W1s reversed", C, "a += (double)w[d + t] * S[(int64_t)i * k + t];",
     "a += (double)w[d + k - 1 - t] * S[(int64_t)i * k + t];"),
    ("no score features", C, "for (int32_t t = 0; t < k; ++t) a += (double)w[d + t] * S[(int64_t)i * k + t];", ""),
    ("W1x unrounded", C, "a += orc_bf16(w[l]) * orc_bf16(X[(int64_t)i * d + l]);",
     "a += (double)w[l] * orc_bf16(X[(int64_t)i * d + l]);"),
    ("W2 transposed index", C, "z += (double)W2[(int64_t)v * H + j] * h[j];", "z += (double)W2[(int64_t)j * L + v] * h[j];"),
    # O6-O10 assignment
    ("gate strict", C, "int adm = (v == 0) || (opts[v].k_skip == 0) || (s1[i] >= (double)opts[v].sim_gate);",
     "int adm = (v == 0) || (opts[v].k_skip == 0) || (s1[i] > (double)opts[v].sim_gate);"),
    ("option 0 gated", C, "int adm = (v == 0) || (opts[v].k_skip == 0) ||", "int adm = (opts[v].k_skip == 0) ||"),
    ("K=0 options gated", C, "int adm = (v == 0) || (opts[v].k_skip == 0) ||", "int adm = (v == 0) ||"),
    ("compliance strict", C, "if (adm && rhat[(int64_t)i * L + v] >= d64) Cm[i] |= 1u << v;",
     "if (adm && rhat[(int64_t)i * L + v] > d64) Cm[i] |= 1u << v;"),
    ("compliance ignores gates", C, "if (adm && rhat[(int64_t)i * L + v] >= d64)", "if (rhat[(int64_t)i * L + v] >= d64)"),
    ("preference slower first", C, "if (x->pth != y->pth) return x->pth > y->pth ? -1 : 1;",
     "if (x->pth != y->pth) return x->pth < y->pth ? -1 : 1;"),
    ("preference higher index", C, "return x->v < y->v ? -1 : (x->v > y->v);                /* lower index",
     "return x->v > y->v ? -1 : (x->v < y->v);                /* lower index"),
    ("preference quality asc", C, "if (x->r != y->r) return x->r > y->r ? -1 : 1;", "if (x->r != y->r) return x->r < y->r ? -1 : 1;"),
    ("priority |C| desc", C, "if (x->c != y->c) return x->c < y->c ? -1 : 1;", "if (x->c != y->c) return x->c > y->c ? -1 : 1;"),
    ("priority i desc", C, "return x->i < y->i ? -1 : (x->i > y->i);                /* i asc",
     "return x->i > y->i ? -1 : (x->i < y->i);                /* i asc"),
    ("quota off by one", C, "if (rem[v] > 0) { a = v; rem[v] -= 1; break; }", "if (rem[v] >= 0) { a = v; rem[v] -= 1; break; }"),
    ("quota never consumed", C, "if (rem[v] > 0) { a = v; rem[v] -= 1; break; }", "if (rem[v] > 0) { a = v; break; }"),
    ("overflow to first preference", C, "if (a < 0) { a = 0; status_out[i]", "if (a < 0) { a = P[(int64_t)i * L]; status_out[i]"),
    ("noncompliant flag <=", C, "if (rhat[(int64_t)i * L + a] < d64) status_out[i] |= ST_NONCOMPLIANT;",
     "if (rhat[(int64_t)i * L + a] <= d64) status_out[i] |= ST_NONCOMPLIANT;"),
    ("gated-all without gates", C, "status_out[i] = (any_gate && n_gate_pass == 0) ? ST_GATED_ALL : 0;",
     "status_out[i] = (n_gate_pass == 0) ? ST_GATED_ALL : 0;"),
    ("largest remainder ties to higher v", C, "if (frac[v] >= 0.0 && (best < 0 || frac[v] > frac[best])) best = v;",
     "if (frac[v] >= 0.0 && (best < 0 || frac[v] >= frac[best])) best = v;"),
    ("largest remainder repeat unit", C, "frac[best] = -1.0; /* each", "/* each"),
    ("largest remainder smallest part", C, "if (frac[v] >= 0.0 && (best < 0 || frac[v] > frac[best])) best = v;",
     "if (frac[v] >= 0.0 && (best < 0 || frac[v] < frac[best])) best = v;"),
    # F1 control plane
    ("o_i slowest", PY, "key = (float(p_th[v]), r, -v)", "key = (-float(p_th[v]), r, -v)"),
    ("o_i ties to lower quality", PY, "key = (float(p_th[v]), r, -v)", "key = (float(p_th[v]), -r, -v)"),
    ("o_i ties to higher v", PY, "key = (float(p_th[v]), r, -v)", "key = (float(p_th[v]), r, v)"),
    ("o_i ignores compliance", PY, "        if r < d64:\n            continue\n        key", "        key"),
    ("ODA excess to faster level", PY, "move(i, i - 1, h[i] - F[i])", "move(i, min(n - 1, i + 1), h[i] - F[i])"),
    ("ODA pull from faster", PY, "shift = min(h[i - m], F[i] - h[i])   # line 10\n                move(i - m, i, shift)",
     "shift = min(h[i - m], F[i] - h[i])   # line 10\n                move(i - m, i, shift * 0.5)"),
    ("ODA slow to fast order", PY, "for i in range(n - 1, -1, -1):          # line 2", "for i in range(n):          # line 2"),
    ("Eq.2 all pairs", PY, "            if p_th[j] > p_th[i]:\n                dq +=", "            if True:\n                dq +="),
    ("Eq.2 transposed D", PY, "dq += P[i][j] * H[i] * D[j][i]", "dq += P[i][j] * H[i] * D[i][j]"),
    ("Philox x1 instead of x0", PY, "(seed & M32, (seed >> 32) & M32))[0]", "(seed & M32, (seed >> 32) & M32))[1]"),
    ("Philox counter words swapped", PY, "philox4x32_10((i, batch_seq & M32,", "philox4x32_10((batch_seq & M32, i,"),
    ("PASM u <= cdf", PY, "if u < cdf_row[j]:", "if u <= cdf_row[j]:"),
    ("uniform from low bits", PY, "np.float32((x0 >> 8) * (1.0 / 16777216.0))", "np.float32((x0 & 0xFFFFFF) * (1.0 / 16777216.0))"),
    ("gate fallback to faster", PY, "        while not (adm >> a) & 1:\n            a -= 1",
     "        while not (adm >> a) & 1:\n            a = (a + 1) % len(opts)"),
    ("PASM sampled from the assigned row", PY, "a = pasm_sample(P[oi], cdf[oi],", "a = pasm_sample(P[0], cdf[0],"),
    ("affinity window off by one", PY, "for o in list(optimal_history)[-window:]:", "for o in list(optimal_history)[-window + 1:]:"),
    ("Eq.3 argmax", PY, "if best is None or cost < best[0]:\n                best = (cost, w)\n        if best is not None:",
     "if best is None or cost > best[0]:\n                best = (cost, w)\n        if best is not None:"),
    ("Eq.3 ties to the highest worker", PY, "if best is None or cost < best[0]:\n                best = (cost, w)\n        if best is not None:",
     "if best is None or cost <= best[0]:\n                best = (cost, w)\n        if best is not None:"),
    ("Eq.3 queue not advanced", PY, "            q[best[1]] += 1\n", ""),
    ("Eq.3 cost without queue", PY, "cost = np.float32(np.float32(q[w]) * np.float32(t_proc[w]))", "cost = np.float32(t_proc[w])"),
    ("Eq.1 objective without Q", PY, "                num += Q[v] * Y[v]", "                num += Y[v]"),
]


def run_pins():
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_oracle_pins.py", "tests/test_oracle_control.py", "tests/test_control_host.py"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    return r.returncode == 0, (r.stdout.strip().splitlines() or [""])[-1]


def rebuild():
    r = subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    return r.returncode == 0, r.stderr[-500:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    backup = {}
    for f in (C, PY):
        backup[f] = open(os.path.join(ROOT, f)).read()
    survived, killed, invalid = [], [], []
    try:
        for name, f, old, new in MUTANTS:
            if args.only and args.only not in name:
                continue
            src = backup[f]
            if src.count(old) != 1:
                invalid.append(name)
                print(f"INVALID  {name} (pattern found {src.count(old)} times)", flush=True)
                continue
            with open(os.path.join(ROOT, f), "w") as fh:
                fh.write(src.replace(old, new))
            if f == C:
                ok, err = rebuild()
                if not ok:
                    invalid.append(name)
                    print(f"NOBUILD  {name}: {err}", flush=True)
                    continue
            passed, last = run_pins()
            (survived if passed else killed).append(name)
            print(f"{'SURVIVED' if passed else 'killed  '} {name}   [{last}]", flush=True)
            with open(os.path.join(ROOT, f), "w") as fh:
                fh.write(src)
    finally:
        for f, src in backup.items():
            with open(os.path.join(ROOT, f), "w") as fh:
                fh.write(src)
        rebuild()
    print(json.dumps({"mutants": len(survived) + len(killed), "killed": len(killed), "survived": survived,
                      "invalid": invalid}))


if __name__ == "__main__":
    main()
