"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is the ONLY code the two sides share.  It draws random numbers and
lays out option tables; it contains none of the method's arithmetic (no cosine,
no top-k, no MLP, no compliance / preference / assignment, no quota rounding).
Every recipe below is stated in DESIGN.md §"Input recipe".

Shapes follow BASELINE.json ``configs`` (C1..C5) and SURVEY.md §8(d):

* embeddings: "unit-norm random embeddings with clustered prompt repeats"
  (BASELINE.json north_star; DiffusionDB-like repeats);
* batch sizes: a 2-state Markov-modulated Poisson process shaped like the
  Twitter trace (SPEC.md S:127-135 describes the bursty generator);
* option tables: {model} x {K} with AC latency (T-K)/T * base + overhead
  ("reducing latency by a factor of (N - K)/N") and
  P_th = floor(60 / latency);
* MLP weights: seeded uniform draws (no trained weights exist).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

T_STEPS = 50            # denoising steps, "N = 50"
AC_OVERHEAD_S = 0.05    # nominal retrieval overhead
CHUNK = 1 << 16         # cache rows are generated in fixed chunks (determinism)

# Base latencies on A100 (Table 2; SD-XL 4.2 s also P:393).
MODEL_LATENCY_S = {
    "SD-XL": 4.2,
    "SD-2.1": 3.84,   # SD-2.1 ~ SD-1.5 latency (Table 2 lists SD1.5 3.84 s)
    "SD-Small": 2.75,
    "Tiny-SD": 2.18,
}
MODEL_ID = {"SD-XL": 0, "SD-2.1": 1, "SD-Small": 2, "Tiny-SD": 3}
# Proposed similarity gates per skip level (unpinned).
GATE_FOR_K = {0: float("-inf"), 5: 0.70, 10: 0.75, 15: 0.80, 20: 0.85, 25: 0.90}


@dataclass
class Config:
    name: str
    N: int                 # batch size (fixed) or max batch for bursty configs
    d: int
    M: int
    k: int
    models: tuple
    ks: tuple
    hidden: int = 256
    bursty: bool = False
    seed: int = 101
    frac_base: float = 1.2     # F_v proportional to frac_base**v
    stress: bool = False       # C5 quota-stress b2 skew
    gpus: tuple = (1,)
    note: str = ""

    @property
    def L(self) -> int:
        return len(self.models) * len(self.ks)


CONFIGS = {
    "C1": Config("C1", 64, 768, 4096, 4, ("SD-XL", "SD-2.1", "Tiny-SD"), (0, 25), seed=101,
                 note="N=64 prompts, d=768, M=4096 cached embeddings, k=4, L=6"),
    "C2": Config("C2", 512, 768, 1_000_000, 4, ("SD-XL", "Tiny-SD"), (0, 5, 10, 15, 20, 25),
                 bursty=True, seed=102,
                 note="Twitter-trace-shaped bursty batches N=16..512, M=1M cache, L=12, single B200"),
    "C3": Config("C3", 256, 768, 10_000_000, 4, ("SD-XL", "Tiny-SD"), (0, 5, 10, 15, 20, 25),
                 seed=103, gpus=(1, 2, 4, 8),
                 note="SYSTEM-X-like steady load N=256, M=10M cache sharded over 8 B200"),
    "C4": Config("C4", 8192, 1024, 4_000_000, 4, ("SD-XL", "SD-2.1", "SD-Small", "Tiny-SD"),
                 (0, 5, 10, 15), seed=104, gpus=(1, 2, 4, 8),
                 note="large-batch tensor-core regime N=8192, M=4M, d=1024, L=16"),
    "C5": Config("C5", 4096, 768, 2_000_000, 4, ("SD-XL", "SD-2.1", "SD-Small", "Tiny-SD"),
                 (0, 5, 10, 15, 20, 25), seed=105, frac_base=1.5, stress=True,
                 note="quota-stress: skewed quality predictions, N=4096, M=2M, L=24"),
}


# --------------------------------------------------------------------------------------
# option table
# --------------------------------------------------------------------------------------
def option_table(models, ks):
    """Options {model} x {K}, ordered slow -> fast (level index 0 = slowest).

    Returns a list of dicts with the argus_option fields (model_id, k_skip,
    p_th_qpm, sim_gate) plus the latency used to order them.  Ties in latency are
    broken by (model order, K) so the order is total.
    """
    rows = []
    for mi, m in enumerate(models):
        for K in ks:
            lat = (T_STEPS - K) / T_STEPS * MODEL_LATENCY_S[m] + AC_OVERHEAD_S
            rows.append(dict(model=m, model_id=MODEL_ID[m], k_skip=int(K),
                             latency_s=lat, p_th_qpm=float(math.floor(60.0 / lat)),
                             sim_gate=GATE_FOR_K.get(int(K), 0.9), _mi=mi))
    rows.sort(key=lambda r: (-r["latency_s"], r["_mi"], r["k_skip"]))
    # the full model (slowest, K=0) must lead; p_th must be non-decreasing
    for a, b in zip(rows, rows[1:]):
        if b["p_th_qpm"] < a["p_th_qpm"]:
            b["p_th_qpm"] = a["p_th_qpm"]
    for r in rows:
        del r["_mi"]
    return rows


def option_arrays(opts):
    """Columnar view: (model_id i32[L], k_skip i32[L], p_th f32[L], sim_gate f32[L])."""
    return (np.array([o["model_id"] for o in opts], np.int32),
            np.array([o["k_skip"] for o in opts], np.int32),
            np.array([o["p_th_qpm"] for o in opts], np.float32),
            np.array([o["sim_gate"] for o in opts], np.float32))


def load_fractions(L, base):
    """Allocator load shares F(v) (Eq. 1 output), here F_v ∝ base**v."""
    f = np.array([base ** v for v in range(L)], np.float64)
    return f / f.sum()


# --------------------------------------------------------------------------------------
# embeddings
# --------------------------------------------------------------------------------------
def _normalize(a):
    n = np.sqrt(np.einsum("ij,ij->i", a, a, dtype=np.float64))
    n[n == 0] = 1.0
    return (a / n[:, None].astype(a.dtype)).astype(np.float32)


class CacheGen:
    """Clustered unit-norm cache embeddings, generated deterministically per chunk.

    n_c = max(16, M // 64) centres mu ~ normalize(N(0, I_d)); cluster popularity
    ~ Zipf(1.1); row = normalize(mu_c + 0.5 g / sqrt(d)) (intra-cluster cos ~ 0.8);
    5 % of rows are exact copies of an earlier row of the same chunk.
    """

    def __init__(self, M: int, d: int, seed: int):
        self.M, self.d, self.seed = int(M), int(d), int(seed)
        self.n_c = max(16, self.M // 64)
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0xC0FFEE])))
        # centres: twice as many as cached clusters; the upper half is "uncached"
        self.centres = _normalize(rng.standard_normal((2 * self.n_c, d), dtype=np.float32))
        p = 1.0 / np.arange(1, self.n_c + 1, dtype=np.float64) ** 1.1
        self.pop = p / p.sum()

    def n_chunks(self):
        return (self.M + CHUNK - 1) // CHUNK

    def chunk(self, ci: int) -> np.ndarray:
        a = ci * CHUNK
        b = min(self.M, a + CHUNK)
        n = b - a
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([self.seed, 1, ci])))
        cl = rng.choice(self.n_c, size=n, p=self.pop)
        g = rng.standard_normal((n, self.d), dtype=np.float32)
        rows = _normalize(self.centres[cl] + np.float32(0.5 / math.sqrt(self.d)) * g)
        dup = rng.random(n) < 0.05
        dup[0] = False
        idx = np.nonzero(dup)[0]
        if idx.size:
            src = (rng.random(idx.size) * idx).astype(np.int64)  # an earlier row in the chunk
            rows[idx] = rows[src]
        return rows

    def chunks(self):
        for ci in range(self.n_chunks()):
            yield ci * CHUNK, self.chunk(ci)

    def all(self, threads: int = 1) -> np.ndarray:
        """All M rows.  threads > 1 generates chunks concurrently (each chunk has its
        own seeded stream, so the result does not depend on `threads`)."""
        out = np.empty((self.M, self.d), np.float32)

        def fill(ci):
            c = self.chunk(ci)
            out[ci * CHUNK:ci * CHUNK + c.shape[0]] = c

        if threads <= 1:
            for ci in range(self.n_chunks()):
                fill(ci)
        else:
            import concurrent.futures as cf
            with cf.ThreadPoolExecutor(max_workers=threads) as ex:
                list(ex.map(fill, range(self.n_chunks())))
        return out

    def rows_at(self, ids) -> np.ndarray:
        ids = np.asarray(ids, np.int64)
        out = np.empty((ids.size, self.d), np.float32)
        for ci in np.unique(ids // CHUNK):
            c = self.chunk(int(ci))
            sel = np.nonzero(ids // CHUNK == ci)[0]
            out[sel] = c[ids[sel] - ci * CHUNK]
        return out


def queries(cache: CacheGen, N: int, seed: int, batch: int = 0, cache_rows=None) -> np.ndarray:
    """N prompts: 30 % exact repeats of a cached row, 50 % fresh members of a
    cached cluster (near hit), 20 % members of an uncached cluster (miss)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 2, batch])))
    d = cache.d
    u = rng.random(N)
    kind = np.where(u < 0.3, 0, np.where(u < 0.8, 1, 2))
    out = np.empty((N, d), np.float32)
    rep = np.nonzero(kind == 0)[0]
    if rep.size:
        ids = rng.integers(0, cache.M, size=rep.size)
        out[rep] = cache_rows[ids] if cache_rows is not None else cache.rows_at(ids)
    near = np.nonzero(kind == 1)[0]
    if near.size:
        cl = rng.choice(cache.n_c, size=near.size, p=cache.pop)
        g = rng.standard_normal((near.size, d), dtype=np.float32)
        out[near] = _normalize(cache.centres[cl] + np.float32(0.5 / math.sqrt(d)) * g)
    miss = np.nonzero(kind == 2)[0]
    if miss.size:
        cl = cache.n_c + rng.integers(0, cache.n_c, size=miss.size)
        g = rng.standard_normal((miss.size, d), dtype=np.float32)
        out[miss] = _normalize(cache.centres[cl] + np.float32(0.5 / math.sqrt(d)) * g)
    return out


def bursty_sizes(n_batches: int, seed: int = 2018, lo: int = 16, hi: int = 512):
    """Twitter-shaped batch sizes: 2-state MMPP, N ~ Poisson(48) (low) /
    Poisson(320) (high), mean dwell 20 / 5 batches, clipped to [lo, hi]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    state, out = 0, []
    for _ in range(n_batches):
        lam = 48 if state == 0 else 320
        out.append(int(min(hi, max(lo, rng.poisson(lam)))))
        if rng.random() < (1 / 20 if state == 0 else 1 / 5):
            state ^= 1
    return out


# --------------------------------------------------------------------------------------
# predictor weights
# --------------------------------------------------------------------------------------
def _logit(q):
    return math.log(q / (1 - q))


def mlp_weights(d: int, k: int, H: int, L: int, seed: int = 7, stress: bool = False):
    """W1 [H][d+k], b1 [H], W2 [L][H], b2 [L] as fp32 (recipe: DESIGN.md).

    W1x ~ U(-sqrt3, sqrt3) (unit variance, so W1x.x ~ N(0,1) for unit x);
    W1s ~ U(-1, 1); b1 ~ U(-.5, .5); W2 ~ U(-a, a) with a = sqrt(3 / (0.7 H)) so that
    W2.h has unit spread; b2_v = logit(q_v), q linear 0.99 -> 0.80 over v.
    stress (C5): options 1 and 2 get b2 = logit(0.999) so ~80 % of prompts rank
    them first among non-full options.
    """
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 3])))
    s3 = math.sqrt(3.0)
    W1 = np.empty((H, d + k), np.float32)
    W1[:, :d] = rng.uniform(-s3, s3, (H, d)).astype(np.float32)
    W1[:, d:] = rng.uniform(-1.0, 1.0, (H, k)).astype(np.float32)
    b1 = rng.uniform(-0.5, 0.5, H).astype(np.float32)
    a = math.sqrt(3.0 / (0.7 * H))
    W2 = rng.uniform(-a, a, (L, H)).astype(np.float32)
    q = np.linspace(0.99, 0.80, L) if L > 1 else np.array([0.99])
    b2 = np.array([_logit(x) for x in q], np.float32)
    if stress and L >= 3:
        b2[1] = b2[2] = np.float32(_logit(0.999))
    return W1, b1, W2, b2


@dataclass
class Problem:
    """A fully materialised small problem (used by tests and the smoke check)."""
    cfg: Config
    cache: np.ndarray
    X: np.ndarray
    opts: list
    W1: np.ndarray
    b1: np.ndarray
    W2: np.ndarray
    b2: np.ndarray
    fractions: np.ndarray
    k: int = 4
    extra: dict = field(default_factory=dict)


def small_problem(name="C1", N=None, M=None, d=None, k=None, seed=None, gates=True,
                  batch=0, stress=None) -> Problem:
    cfg = CONFIGS[name]
    N = cfg.N if N is None else N
    M = cfg.M if M is None else M
    d = cfg.d if d is None else d
    k = cfg.k if k is None else k
    seed = cfg.seed if seed is None else seed
    stress = cfg.stress if stress is None else stress
    cg = CacheGen(M, d, seed) if M > 0 else None
    cache = cg.all() if cg is not None else np.zeros((0, d), np.float32)
    if cg is not None:
        X = queries(cg, N, seed, batch, cache_rows=cache)
    else:
        X = _normalize(np.random.Generator(np.random.PCG64(seed)).standard_normal((N, d), dtype=np.float32))
    opts = option_table(cfg.models, cfg.ks)
    if not gates:
        for o in opts:
            o["sim_gate"] = float("-inf")
    L = len(opts)
    W1, b1, W2, b2 = mlp_weights(d, k, cfg.hidden, L, stress=stress)
    return Problem(cfg, cache, X, opts, W1, b1, W2, b2, load_fractions(L, cfg.frac_base), k=k)
