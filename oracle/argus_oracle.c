/*
 * argus_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the ARGUS routing
 * hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load or execute it.  It
 * shares no code, header, table or helper with the CUDA path in
 * paper_2511_06724_b200/ (it does not include include/argus.h), and the CUDA path
 * never loads it.
 *
 * Citations (PAPER.md line P:<n>, SPEC.md line S:<n>):
 *   O1  canonical inputs: fp32 -> bf16 round-to-nearest-even
 *   O2  norms            ||x|| = sqrt(sum x^2)                       ("similarity search")
 *   O3  cosine           s_ij = <x_i,c_j> / (||x_i|| ||c_j||)
 *   O4  top-k            k largest (s desc, global id asc)            ("most similar")
 *   O5  predictor        r = sigmoid(W2 relu(W1 [x;s] + b1) + b2), r_0 := 1
 *   O6  gates            A_i = {v : v = 0 or k_skip_v = 0 or s_i1 >= tau_v}
 *   O7  compliance       C_i = {v in A_i : r_iv >= delta}, delta = 0.9
 *   O8  preference       pi_i = A_i sorted by (r desc, p_th desc, v asc)
 *   O9  priority         prompts sorted by (|C_i| asc, i asc)
 *   O10 serial dictatorship under per-option quotas, overflow -> option 0
 *   quotas               largest remainder of F*N                   (P:289 F(v))
 *
 * Every floating-point value is carried in double.  The only float arithmetic is
 * the bf16 rounding of the inputs (an exact bit operation) and the widening of
 * fp32 parameters.
 *
 * Parity pins live in tests/test_oracle_*.py (closed forms, brute force,
 * invariants, the S:67 worked example, the P-ODA monotone special case).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t model_id;
    int32_t k_skip;
    float p_th_qpm;
    float sim_gate;
} orc_option; /* same field order as the boundary's option record */

#define ORC_OK 0
#define ORC_OVERFLOW 1
#define ORC_EINVAL (-1)

#define ST_OVERFLOW 1u
#define ST_NONCOMPLIANT 2u
#define ST_GATED_ALL 4u

/* ---------------------------------------------------------------- O1: bf16 RNE */
/* Round an fp32 value to the nearest bf16 (ties to even) and return it as double.
 * bf16 keeps the top 16 bits of the fp32 pattern.  NaN/Inf are passed through
 * (the boundary rejects them before they reach here). */
double orc_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return (double)x;
    uint32_t lower = u & 0xffffu;
    uint32_t upper = u >> 16;
    if (lower > 0x8000u || (lower == 0x8000u && (upper & 1u))) upper += 1u;
    uint32_t r = upper << 16;
    float f;
    memcpy(&f, &r, 4);
    return (double)f;
}

void orc_bf16_array(const float* in, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_bf16(in[i]);
}

/* ---------------------------------------------------------------- O2/O3: cosine */
static double dot_bf16(const float* a, const float* b, int32_t d) {
    double s = 0.0;
    for (int32_t l = 0; l < d; ++l) s += orc_bf16(a[l]) * orc_bf16(b[l]);
    return s;
}

static double norm_bf16(const float* a, int32_t d) { return sqrt(dot_bf16(a, a, d)); }

/* cos(x_i, c_j) for one pair, O3, in fp64 over the bf16 values. */
double orc_cosine(const float* x, const float* c, int32_t d) {
    double nx = norm_bf16(x, d), nc = norm_bf16(c, d);
    if (nx == 0.0 || nc == 0.0) return NAN;
    return dot_bf16(x, c, d) / (nx * nc);
}

/* O3 for every pair: S[i][j] = cos(x_i, c_j) in fp64 over the bf16 values (the full
 * N x M matrix, for element-wise parity of the GPU's captured scores, T1/T2). */
int orc_score_matrix(const float* X, int32_t N, const float* C, int64_t M, int32_t d, int nthreads, double* S) {
    if (N < 0 || M < 0 || d <= 0) return ORC_EINVAL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int32_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < M; ++j) S[(int64_t)i * M + j] = orc_cosine(X + (int64_t)i * d, C + j * d, d);
    return ORC_OK;
}

/* ---------------------------------------------------------------- O4: top-k */
/* (s, g) beats (s', g') iff s > s' or (s == s' and g < g').  Ties go to the
 * older (lower-id) cache entry. */
static int better(double s, uint32_t g, double s2, uint32_t g2) {
    return s > s2 || (s == s2 && g < g2);
}

/* O4 step: insert (s, g) into the sorted best-k list bs/bg holding *filled entries. */
static void topk_insert(double s, uint32_t g, int32_t k, int* filled, double* bs, uint32_t* bg) {
    if (*filled < k || better(s, g, bs[k - 1], bg[k - 1])) {
        int p = *filled < k ? (*filled)++ : k - 1;
        while (p > 0 && better(s, g, bs[p - 1], bg[p - 1])) {
            bs[p] = bs[p - 1]; bg[p] = bg[p - 1]; --p;
        }
        bs[p] = s; bg[p] = g;
    }
}

/* For each prompt: the k best (s, g) over all cache rows, sorted best first.
 * Rows beyond M pad with (score -1, id 0xFFFFFFFF).  ids[j] is the global id of
 * row j (NULL -> j).  Returns ORC_EINVAL on zero-norm / non-finite input. */
int orc_scan_topk(const float* X, int32_t N, const float* C, int64_t M, int32_t d, int32_t k,
                  const uint32_t* ids, int nthreads, double* topk_score, uint32_t* topk_idx) {
    if (N < 0 || M < 0 || d <= 0 || k <= 0) return ORC_EINVAL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    /* O1 once per input: the bf16 values of X and C (exactly representable in float,
     * so this copy is lossless); the products and sums below are the same fp64
     * operations in the same order as dot_bf16 on the raw rows. */
    float* Cb = (float*)malloc(sizeof(float) * (size_t)(M > 0 ? M : 1) * (size_t)d);
    float* Xb = (float*)malloc(sizeof(float) * (size_t)(N > 0 ? N : 1) * (size_t)d);
    double* nc = (double*)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
    if (!Cb || !Xb || !nc) { free(Cb); free(Xb); free(nc); return ORC_EINVAL; }
    int bad = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(|: bad)
#endif
    for (int64_t j = 0; j < M; ++j) {
        for (int32_t l = 0; l < d; ++l) Cb[j * d + l] = (float)orc_bf16(C[j * d + l]);
        /* O2: norm of the bf16 cache row */
        double q = 0.0;
        for (int32_t l = 0; l < d; ++l) q += (double)Cb[j * d + l] * (double)Cb[j * d + l];
        nc[j] = sqrt(q);
        if (!(nc[j] > 0.0) || !isfinite(nc[j])) bad = 1;
    }
    for (int64_t e = 0; e < (int64_t)N * d; ++e) Xb[e] = (float)orc_bf16(X[e]);
    if (bad) { free(Cb); free(Xb); free(nc); return ORC_EINVAL; }
    int badq = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) reduction(|: badq)
#endif
    for (int32_t i = 0; i < N; ++i) {
        const float* x = Xb + (int64_t)i * d;
        double* bs = topk_score + (int64_t)i * k;
        uint32_t* bg = topk_idx + (int64_t)i * k;
        double nx = 0.0;
        for (int32_t l = 0; l < d; ++l) nx += (double)x[l] * (double)x[l];
        nx = sqrt(nx);                                               /* O2 */
        for (int32_t t = 0; t < k; ++t) { bs[t] = -1.0; bg[t] = 0xFFFFFFFFu; }
        if (!(nx > 0.0) || !isfinite(nx)) { badq = 1; continue; }
        int filled = 0;
        for (int64_t j = 0; j < M; ++j) {
            const float* c = Cb + j * d;
            double dot = 0.0;
            for (int32_t l = 0; l < d; ++l) dot += (double)x[l] * (double)c[l];
            double s = dot / (nx * nc[j]);                           /* O3 */
            uint32_t g = ids ? ids[j] : (uint32_t)j;
            topk_insert(s, g, k, &filled, bs, bg);                  /* O4 */
        }
    }
    free(Cb); free(Xb); free(nc);
    return badq ? ORC_EINVAL : ORC_OK;
}

/* O4 alone on given scores S [N][M] (row stride ld; parity test T2 replays it on
 * the GPU's own fp32 scores): the k best (s, g) per row, sorted
 * best first, padded like orc_scan_topk.  ids[j] is the global id of column j. */
int orc_topk_of_scores(const double* S, int32_t N, int64_t M, int64_t ld, int32_t k, const uint32_t* ids,
                       double* topk_score, uint32_t* topk_idx) {
    if (N < 0 || M < 0 || ld < M || k <= 0) return ORC_EINVAL;
    for (int32_t i = 0; i < N; ++i) {
        double* bs = topk_score + (int64_t)i * k;
        uint32_t* bg = topk_idx + (int64_t)i * k;
        for (int32_t t = 0; t < k; ++t) { bs[t] = -1.0; bg[t] = 0xFFFFFFFFu; }
        int filled = 0;
        for (int64_t j = 0; j < M; ++j)
            topk_insert(S[(int64_t)i * ld + j], ids ? ids[j] : (uint32_t)j, k, &filled, bs, bg);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- O5: predictor */
/* h = max(0, W1x.bf16(x) + W1s.s + b1);  r = 1 / (1 + exp(-(W2 h + b2)));  r_0 := 1.
 * W1 is [H][d+k] row-major: columns [0,d) act on the embedding (rounded to bf16,
 * the canonical tensor-core operand), columns [d,d+k) on the top-k scores. */
int orc_mlp(const float* X, const double* S, int32_t N, int32_t d, int32_t k, int32_t H, int32_t L,
            const float* W1, const float* b1, const float* W2, const float* b2, int nthreads,
            double* rhat) {
    if (N < 0 || d <= 0 || k < 0 || H <= 0 || L <= 0) return ORC_EINVAL;  /* k = 0: SM-mode classifier */
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int32_t i = 0; i < N; ++i) {
        double* h = (double*)malloc(sizeof(double) * (size_t)H);
        for (int32_t j = 0; j < H; ++j) {
            const float* w = W1 + (int64_t)j * (d + k);
            double a = 0.0;
            for (int32_t l = 0; l < d; ++l) a += orc_bf16(w[l]) * orc_bf16(X[(int64_t)i * d + l]);
            for (int32_t t = 0; t < k; ++t) a += (double)w[d + t] * S[(int64_t)i * k + t];
            a += (double)b1[j];
            h[j] = a > 0.0 ? a : 0.0;
        }
        for (int32_t v = 0; v < L; ++v) {
            double z = (double)b2[v];
            for (int32_t j = 0; j < H; ++j) z += (double)W2[(int64_t)v * H + j] * h[j];
            rhat[(int64_t)i * L + v] = 1.0 / (1.0 + exp(-z));
        }
        rhat[(int64_t)i * L + 0] = 1.0; /* the full model is the reference */
        free(h);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- O6..O10: assignment */
typedef struct { double r; double pth; int32_t v; } pref_key;

static int pref_cmp(const void* a, const void* b) {
    const pref_key* x = (const pref_key*)a;
    const pref_key* y = (const pref_key*)b;
    if (x->r != y->r) return x->r > y->r ? -1 : 1;          /* quality desc   */
    if (x->pth != y->pth) return x->pth > y->pth ? -1 : 1;  /* faster first   */
    return x->v < y->v ? -1 : (x->v > y->v);                /* lower index    */
}

typedef struct { int32_t c; int32_t i; } prio_key;

static int prio_cmp(const void* a, const void* b) {
    const prio_key* x = (const prio_key*)a;
    const prio_key* y = (const prio_key*)b;
    if (x->c != y->c) return x->c < y->c ? -1 : 1;          /* |C_i| asc */
    return x->i < y->i ? -1 : (x->i > y->i);                /* i asc     */
}

/* rhat [N][L] (double; the oracle's own or the GPU's fp32 values widened),
 * s1 [N] top-1 similarity, quota [L] >= 0, delta compared as (double)(float)delta.
 * Outputs: option_out [N], status_out [N]; optional (may be NULL): adm_mask [N],
 * cmp_mask [N], pref [N][L] (0xFF past |A_i|), order [N] (priority order). */
int orc_assign(const double* rhat, const double* s1, int32_t N, int32_t L, const orc_option* opts,
               const int32_t* quota, float delta, int32_t* option_out, uint8_t* status_out,
               uint32_t* adm_mask, uint32_t* cmp_mask, uint8_t* pref, int32_t* order) {
    if (N < 0 || L <= 0 || L > 32) return ORC_EINVAL;
    const double d64 = (double)delta;
    uint32_t* A = (uint32_t*)calloc((size_t)(N > 0 ? N : 1), 4);
    uint32_t* Cm = (uint32_t*)calloc((size_t)(N > 0 ? N : 1), 4);
    uint8_t* P = (uint8_t*)malloc((size_t)(N > 0 ? N : 1) * (size_t)L);
    prio_key* pk = (prio_key*)malloc(sizeof(prio_key) * (size_t)(N > 0 ? N : 1));
    int32_t* nA = (int32_t*)calloc((size_t)(N > 0 ? N : 1), 4);
    int32_t* rem = (int32_t*)malloc(sizeof(int32_t) * (size_t)L);
    int any_gate = 0;
    for (int32_t v = 0; v < L; ++v) if (opts[v].k_skip != 0) any_gate = 1;
    for (int32_t i = 0; i < N; ++i) {
        int n_gate_pass = 0;
        for (int32_t v = 0; v < L; ++v) {
            /* O6: gates -- option 0 and K=0 options are never gated */
            int adm = (v == 0) || (opts[v].k_skip == 0) || (s1[i] >= (double)opts[v].sim_gate);
            if (opts[v].k_skip != 0 && s1[i] >= (double)opts[v].sim_gate) ++n_gate_pass;
            if (adm) A[i] |= 1u << v;
            /* O7: compliance */
            if (adm && rhat[(int64_t)i * L + v] >= d64) Cm[i] |= 1u << v;
        }
        /* O8: preference order over A_i */
        pref_key ks[32];
        int n = 0;
        for (int32_t v = 0; v < L; ++v)
            if (A[i] >> v & 1u) { ks[n].r = rhat[(int64_t)i * L + v]; ks[n].pth = opts[v].p_th_qpm; ks[n].v = v; ++n; }
        qsort(ks, (size_t)n, sizeof(pref_key), pref_cmp);
        for (int32_t t = 0; t < L; ++t) P[(int64_t)i * L + t] = t < n ? (uint8_t)ks[t].v : 0xFF;
        nA[i] = n;
        /* O9: priority key */
        pk[i].c = __builtin_popcount(Cm[i]);
        pk[i].i = i;
        status_out[i] = (any_gate && n_gate_pass == 0) ? ST_GATED_ALL : 0;
    }
    qsort(pk, (size_t)N, sizeof(prio_key), prio_cmp);
    /* O10: serial dictatorship */
    for (int32_t v = 0; v < L; ++v) rem[v] = quota[v];
    int overflow = 0;
    for (int32_t t = 0; t < N; ++t) {
        int32_t i = pk[t].i;
        int32_t a = -1;
        for (int32_t r = 0; r < nA[i]; ++r) {
            int32_t v = P[(int64_t)i * L + r];
            if (rem[v] > 0) { a = v; rem[v] -= 1; break; }
        }
        if (a < 0) { a = 0; status_out[i] |= ST_OVERFLOW; overflow = 1; }
        if (rhat[(int64_t)i * L + a] < d64) status_out[i] |= ST_NONCOMPLIANT;
        option_out[i] = a;
        if (order) order[t] = i;
    }
    if (adm_mask) memcpy(adm_mask, A, sizeof(uint32_t) * (size_t)N);
    if (cmp_mask) memcpy(cmp_mask, Cm, sizeof(uint32_t) * (size_t)N);
    if (pref) memcpy(pref, P, (size_t)N * (size_t)L);
    free(A); free(Cm); free(P); free(pk); free(nA); free(rem);
    return overflow ? ORC_OVERFLOW : ORC_OK;
}

/* ---------------------------------------------------------------- quotas */
/* Largest remainder: t_v = (f_v * N) / S with S = sum_v f_v (summed v = 0..L-1),
 * c_v = floor(t_v), the N - sum c_v leftover units go to the largest fractional
 * parts t_v - c_v, ties to the lower v.  Sum c = N exactly. */
int orc_quota_from_fractions(const double* f, int32_t L, int32_t N, int32_t* c) {
    if (L <= 0 || N < 0) return ORC_EINVAL;
    double S = 0.0;
    for (int32_t v = 0; v < L; ++v) {
        if (!(f[v] >= 0.0) || !isfinite(f[v])) return ORC_EINVAL;
        S += f[v];
    }
    if (!(S > 0.0)) return ORC_EINVAL;
    double frac[64];
    if (L > 64) return ORC_EINVAL;
    int64_t used = 0;
    for (int32_t v = 0; v < L; ++v) {
        double t = (f[v] * (double)N) / S;
        double fl = floor(t);
        c[v] = (int32_t)fl;
        frac[v] = t - fl;
        used += c[v];
    }
    int64_t left = (int64_t)N - used;
    while (left > 0) {
        int32_t best = -1;
        for (int32_t v = 0; v < L; ++v)
            if (frac[v] >= 0.0 && (best < 0 || frac[v] > frac[best])) best = v;
        c[best] += 1;
        frac[best] = -1.0; /* each option receives at most one leftover unit */
        --left;
    }
    while (left < 0) { /* only reachable through rounding of t; take from the smallest parts */
        int32_t worst = -1;
        for (int32_t v = L - 1; v >= 0; --v)
            if (c[v] > 0 && (worst < 0 || frac[v] < frac[worst])) worst = v;
        c[worst] -= 1;
        frac[worst] = 2.0;
        ++left;
    }
    return ORC_OK;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
