/*
 * kvt_oracle.c -- CPU restatement of the LeoAM / kvtier selection + sparse-attention path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the CUDA path and the
 * CPU baseline timed by bench.py.  Nothing in paper_2506_20187_b200/ may import,
 * link or call it.  Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline
 * and --impl reference legs) use it.
 *
 * Everything here is plain C99 on float64.  It restates, per function:
 *   ora_dot / ora_scores      importance.py:27-33   attention_logits = k.q / sqrt(d)
 *   ora_abstract              importance.py:80-87   make_abstract (elementwise max/min)
 *   ora_bounds                importance.py:108-137 bound_chunk / bound_chunks_batch
 *   ora_topk                  engine.py:338,346 and test_chunk_tree.py:25-28
 *                             (lexsort((arange, -scores))[:k]: score desc, index asc)
 *   ora_part_* (B&B)          chunk_tree.py:171-210 build_partition,
 *                             chunk_tree.py:233-338 select_top_k,
 *                             chunk_tree.py:344-379 merge_desert
 *   ora_runs                  engine.py:176-183     _token_runs
 *   ora_attention             engine.py:145-154     attention_output (+ importance.py:36-43 softmax)
 *   ora_synth_lane            trace.py:270-315      generate_synthetic's planted model, as the
 *                             counter-hash generator of csrc/synth.cu (bench/test inputs)
 *
 * Canonical arithmetic (shared *definition* with the CUDA kernels, written independently):
 *   A dot product over d dims is accumulated in 32 partial sums.  Dim j goes to partial
 *   p[(j >> 2) & 31], each partial is a chain of IEEE fma() in increasing j, and the 32
 *   partials are combined by a fixed tree: p[l] += p[l + 16] (l < 16), then +8, +4, +2, +1.
 *   The token score is fl(dot) / fl(sqrt(d)).  Inputs (f32/bf16/f16 keys, f32 queries) are
 *   exactly representable in f64, so the products are exact and the only roundings are the
 *   chain/tree additions -- which are identical on host and device.
 *   The reference sums with numpy pairwise / BLAS dgemv order; the two agree except at f64
 *   near-ties (~1e-16 relative), which the golden tests check never occur on the
 *   reference's own fixtures.
 *
 * Bounds are made *sound with respect to the canonical scores* by widening the computed
 * upper/lower sums by 2*gamma_n*A, A = sum_j |q_j| max(|max_j|, |min_j|), n = chain length
 * + tree depth (see ora_bound_slack).  Single-row abstracts are exact (no widening), as in
 * the reference (importance.py:114 "Exact ... on singletons"), and so are abstracts whose
 * unwidened U == L (all rows equal; see ora_bounds2).
 *
 * Compile: see oracle/Makefile (-O2 -ffp-contract=off; fma() is the explicit fused op).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <time.h>

#define ORA_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------ */
/* canonical reduction                                                                   */
/* ------------------------------------------------------------------------------------ */

static double tree32(double p[32]) {
    for (int off = 16; off >= 1; off >>= 1)
        for (int l = 0; l < off; ++l) p[l] = p[l] + p[l + off];
    return p[0];
}

ORA_API double ora_dot(const double* q, const double* k, int d) {
    double p[32];
    memset(p, 0, sizeof p);
    for (int j = 0; j < d; ++j) {
        int l = (j >> 2) & 31;
        p[l] = fma(q[j], k[j], p[l]);
    }
    return tree32(p);
}

ORA_API double ora_sqrt_d(int d) { return sqrt((double)d); }

/* Raw canonical dots: the selection key of the B200 pipeline (a positive scale does not
 * change the order; the logit fl(dot)/fl(sqrt d) is only formed for the softmax). */
ORA_API void ora_dots(const double* q, const double* keys, int64_t n, int d, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = ora_dot(q, keys + i * (int64_t)d, d);
}

/* importance.py:27-33 attention_logits, canonical order */
ORA_API void ora_scores(const double* q, const double* keys, int64_t n, int d, double* out) {
    double s = sqrt((double)d);
    for (int64_t i = 0; i < n; ++i) out[i] = ora_dot(q, keys + i * (int64_t)d, d) / s;
}

/* importance.py:80-87 make_abstract over keys[start:end) */
ORA_API void ora_abstract(const double* keys, int d, int64_t start, int64_t end, double* mx, double* mn) {
    for (int j = 0; j < d; ++j) { mx[j] = keys[start * d + j]; mn[j] = mx[j]; }
    for (int64_t i = start + 1; i < end; ++i) {
        const double* r = keys + i * (int64_t)d;
        for (int j = 0; j < d; ++j) {
            if (r[j] > mx[j]) mx[j] = r[j];
            if (r[j] < mn[j]) mn[j] = r[j];
        }
    }
}

/* Chain length of one partial (<= 4*ceil(d/128)) plus tree depth 5. */
static int chain_len(int d) { return 4 * ((d + 127) / 128) + 5; }

ORA_API double ora_bound_slack_factor(int d) { return (double)(2 * chain_len(d) + 4) * 0x1p-53; }

/* importance.py:108-137 bound_chunk / bound_chunks_batch (logit mode), sound canonical form.
 * rows[i] = number of real tokens summarised by abstract i (1 => exact, no widening). */
ORA_API void ora_bounds2(const double* q, const double* mx, const double* mn, int64_t m, int d,
                         const int64_t* rows, double* U, double* L, int scaled) {
    double s = sqrt((double)d);
    double fac = ora_bound_slack_factor(d);
    for (int64_t c = 0; c < m; ++c) {
        const double* M = mx + c * (int64_t)d;
        const double* N = mn + c * (int64_t)d;
        double pu[32], pl[32], pa[32];
        memset(pu, 0, sizeof pu); memset(pl, 0, sizeof pl); memset(pa, 0, sizeof pa);
        for (int j = 0; j < d; ++j) {
            int l = (j >> 2) & 31;
            double qj = q[j];
            double hi = qj >= 0.0 ? M[j] : N[j];
            double lo = qj >= 0.0 ? N[j] : M[j];
            pu[l] = fma(qj, hi, pu[l]);
            pl[l] = fma(qj, lo, pl[l]);
            pa[l] = fma(fabs(qj), fmax(fabs(M[j]), fabs(N[j])), pa[l]);
        }
        double u = tree32(pu), lo = tree32(pl), a = tree32(pa);
        /* U == L before widening: RN fma/add are monotone, so the unwidened chains enclose
         * every canonical dot of the chunk, and equal ends pin them all -- exact, no widening
         * (a chunk of identical rows; the walkthrough's flat chunks, test_chunk_tree.py:214) */
        if ((rows == NULL || rows[c] > 1) && u != lo) {
            double slack = a * fac;
            u = u + slack;
            lo = lo - slack;
        }
        U[c] = scaled ? u / s : u;
        L[c] = scaled ? lo / s : lo;
    }
}

ORA_API void ora_bounds(const double* q, const double* mx, const double* mn, int64_t m, int d,
                        const int64_t* rows, double* U, double* L) {
    ora_bounds2(q, mx, mn, m, d, rows, U, L, 1);
}

/* ------------------------------------------------------------------------------------ */
/* reference-mode bounds: numpy's own arithmetic, for the B&B restatement                */
/* ------------------------------------------------------------------------------------ */

/* numpy DOUBLE_pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), blocksize 128. */
static double np_pairwise(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
    }
}

/* ndarray.sum() over a contiguous run (verified bit-equal to numpy 2.3 in
 * tests/test_oracle_golden.py::test_np_sum_restatement). */
ORA_API double ora_np_sum(const double* a, int64_t n) { return np_pairwise(a, n); }

/* importance.py:108-126 bound_chunk exactly as numpy evaluates it:
 * a = q*max, b = q*min (rounded products), U = sum(maximum(a,b))/sqrt(d), L likewise. */
ORA_API void ora_bounds_ref(const double* q, const double* mx, const double* mn, int64_t m, int d,
                            double* U, double* L) {
    double s = sqrt((double)d);
    double* hi = (double*)malloc(sizeof(double) * 2 * (size_t)d);
    double* lo = hi + d;
    for (int64_t c = 0; c < m; ++c) {
        for (int j = 0; j < d; ++j) {
            double a = q[j] * mx[c * d + j];
            double b = q[j] * mn[c * d + j];
            hi[j] = a > b ? a : b;   /* np.maximum (no NaNs here) */
            lo[j] = a < b ? a : b;
        }
        U[c] = ora_np_sum(hi, d) / s;
        L[c] = ora_np_sum(lo, d) / s;
    }
    free(hi);
}

/* ------------------------------------------------------------------------------------ */
/* INT4 KV codec (north-star item 4; the reference has no quantizer -- parity of the codes */
/* is against this definition)                                         */
/* ------------------------------------------------------------------------------------ */
/* Record per token: d/2 code bytes (dim 2j in the low nibble, 2j+1 in the high nibble),
 * then d/32 (scale, min) fp16 pairs.  Per group of 32 dims (GPU: quant.cu kv_quant_kernel):
 *   lo, hi = min, max of the inputs clamped to the fp16 range
 *   m   = fp16_rd(lo)
 *   s   = fp16_ru(fl_ru(fl_ru(hi - m) * R15)),   R15 = fl_ru(1/15)
 *   inv = fl32(1 / s)
 *   code = s == 0 ? 0 : RN_int(fl32(x - m) * inv)            (ties to even, no clamp needed:
 *          the outward rounding puts the product in [0, 15 (1 + 2^-24)])
 *   x^   = fmaf(code, s, m)                                  (one f32 rounding)
 * RN_int of the exact product is fmaf(a, inv, 1.5 * 2^23) - 1.5 * 2^23.  The directed
 * roundings are built from round-to-nearest operations plus exact error terms, so this
 * file needs no fenv. */

ORA_API int ora_i4_record_bytes(int d) { return d / 2 + (d / 32) * 4; }

static float clamp_h(float x) { return x > 65504.0f ? 65504.0f : (x < -65504.0f ? -65504.0f : x); }

static float sub_ru(float a, float b) {  /* fl_ru(a - b) via TwoSum's exact error */
    volatile float s = a - b;
    volatile float bb = s - a;
    volatile float err = (a - (s - bb)) + (-b - bb);
    return err > 0.0f ? nextafterf(s, INFINITY) : s;
}
static float mul_ru(float a, float b) {  /* fl_ru(a * b): the fma residual is exact */
    volatile float p = a * b;
    float err = fmaf(a, b, -p);
    return err > 0.0f ? nextafterf(p, INFINITY) : p;
}
static uint16_t h_bits(_Float16 h) { uint16_t u; memcpy(&u, &h, 2); return u; }
static _Float16 h_from(uint16_t u) { _Float16 h; memcpy(&h, &u, 2); return h; }
static _Float16 h_next(_Float16 h, int up) {  /* adjacent finite fp16 toward +inf (up) or -inf */
    uint16_t u = h_bits(h);
    if ((u & 0x7fff) == 0) return h_from(up ? 0x0001 : 0x8001);
    int neg = u >> 15;
    return h_from((uint16_t)((neg ^ up) ? u + 1 : u - 1));
}
static _Float16 h_rd(float x) { _Float16 h = (_Float16)x; return (float)h > x ? h_next(h, 0) : h; }
static _Float16 h_ru(float x) { _Float16 h = (_Float16)x; return (float)h < x ? h_next(h, 1) : h; }

ORA_API void ora_i4_quant(const float* x, int64_t n, int d, uint8_t* rec) {
    const int rb = ora_i4_record_bytes(d);
    const float magic = 12582912.0f, r15 = 0.0666666701436042785645f;
    for (int64_t t = 0; t < n; ++t) {
        const float* xt = x + t * d;
        uint8_t* r = rec + t * rb;
        memset(r, 0, (size_t)rb);
        for (int g = 0; g < d / 32; ++g) {
            float lo = clamp_h(xt[32 * g]), hi = lo;
            for (int j = 1; j < 32; ++j) {
                float v = clamp_h(xt[32 * g + j]);
                if (v < lo) lo = v;
                if (v > hi) hi = v;
            }
            _Float16 mh = h_rd(lo);
            float mn = (float)mh;
            _Float16 sh = h_ru(mul_ru(sub_ru(hi, mn), r15));
            float sc = (float)sh;
            volatile float inv = 1.0f / sc;
            for (int j = 0; j < 32; ++j) {
                int c = 0;
                if (sc != 0.0f) {
                    volatile float num = clamp_h(xt[32 * g + j]) - mn;
                    c = (int)(fmaf(num, inv, magic) - magic);
                }
                int dim = 32 * g + j;
                r[dim >> 1] |= (uint8_t)(c << ((dim & 1) * 4));
            }
            memcpy(r + d / 2 + 4 * g, &sh, 2);
            memcpy(r + d / 2 + 4 * g + 2, &mh, 2);
        }
    }
}

ORA_API void ora_i4_dequant(const uint8_t* rec, int64_t n, int d, float* x) {
    const int rb = ora_i4_record_bytes(d);
    for (int64_t t = 0; t < n; ++t) {
        const uint8_t* r = rec + t * rb;
        for (int g = 0; g < d / 32; ++g) {
            _Float16 sh, mh;
            memcpy(&sh, r + d / 2 + 4 * g, 2);
            memcpy(&mh, r + d / 2 + 4 * g + 2, 2);
            float sc = (float)sh, mn = (float)mh;
            for (int j = 0; j < 32; ++j) {
                int dim = 32 * g + j;
                int c = (r[dim >> 1] >> ((dim & 1) * 4)) & 15;
                x[t * d + dim] = fmaf((float)c, sc, mn);
            }
        }
    }
}

/* ------------------------------------------------------------------------------------ */
/* Synthetic lanes (bench / test inputs).  Host restatement of the counter-hash generator
 * defined in paper_2506_20187_b200/csrc/synth.cu (the planted-desert model of
 * trace.py:270-315 generate_synthetic): same hash, same sequence of round-to-nearest f32
 * operations (this file builds with -ffp-contract=off), bf16 round-to-nearest-even.  K and
 * V receive the bf16 values widened to f32, [n, d] each (either may be NULL). */

static uint32_t syn_mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
static uint32_t syn_hash(uint32_t s, uint32_t x) { return syn_mix(syn_mix(x) ^ s); }
static float syn_normal(uint32_t s, uint32_t x) {
    uint32_t h0 = syn_hash(s, 2u * x), h1 = syn_hash(s, 2u * x + 1u);
    uint32_t isum = (h0 & 0xffffu) + (h0 >> 16) + (h1 & 0xffffu) + (h1 >> 16);
    volatile float z = (float)isum * 0x1p-16f;
    z = z - 2.0f;
    return z * 1.7320508075688772f;
}
static float bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;  /* finite inputs only */
    memcpy(&f, &u, 4);
    return f;
}

ORA_API void ora_synth_lane(float* K, float* V, int64_t n, int d, uint32_t lane_seed, const float* u,
                            const int32_t* regions, int R, float desert_base, float desert_span,
                            float hot_base, float hot_span, float noise_scale, int planted) {
    uint32_t s_k = syn_mix(lane_seed ^ 0x9e3779b9u), s_v = syn_mix(lane_seed ^ 0x85ebca6bu);
    uint32_t s_a = syn_mix(lane_seed ^ 0xc2b2ae35u);
    for (int64_t t = 0; t < n; ++t) {
        float a = 0.0f;
        if (planted) {
            int hot = 0;
            for (int r = 0; r < R; ++r) hot |= (t >= regions[2 * r] && t < regions[2 * r + 1]);
            float r24 = (float)(syn_hash(s_a, (uint32_t)t) >> 8) * 0x1p-24f;
            volatile float prod = r24 * (hot ? hot_span : desert_span);
            a = prod + (hot ? hot_base : desert_base);
        }
        for (int j = 0; j < d; ++j) {
            uint32_t x = (uint32_t)(t * d + j);
            if (K) {
                float k = syn_normal(s_k, x);
                if (planted) {
                    volatile float au = a * u[j];
                    volatile float nz = k * noise_scale;
                    k = au + nz;
                }
                K[t * d + j] = bf16_rne(k);
            }
            if (V) V[t * d + j] = bf16_rne(syn_normal(s_v, x));
        }
    }
}

/* ------------------------------------------------------------------------------------ */
/* exact top-k (score desc, index asc)                                                   */
/* ------------------------------------------------------------------------------------ */

typedef struct { double s; int64_t i; } scored_t;

static int cmp_scored(const void* a, const void* b) {
    const scored_t* x = (const scored_t*)a;
    const scored_t* y = (const scored_t*)b;
    if (x->s > y->s) return -1;
    if (x->s < y->s) return 1;
    return (x->i > y->i) - (x->i < y->i);
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* out: the k selected indices, ascending.  Returns k. */
ORA_API int64_t ora_topk(const double* scores, int64_t n, int64_t k, int64_t* out) {
    if (k <= 0) return 0;
    scored_t* t = (scored_t*)malloc(sizeof(scored_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) { t[i].s = scores[i] == 0.0 ? 0.0 : scores[i]; t[i].i = i; }
    qsort(t, (size_t)n, sizeof(scored_t), cmp_scored);
    for (int64_t i = 0; i < k; ++i) out[i] = t[i].i;
    free(t);
    qsort(out, (size_t)k, sizeof(int64_t), cmp_i64);
    return k;
}

/* engine.py:176-183 _token_runs; sel ascending.  Writes starts/ends, returns run count. */
ORA_API int64_t ora_runs(const int64_t* sel, int64_t k, int64_t* starts, int64_t* ends) {
    int64_t r = 0;
    for (int64_t i = 0; i < k; ++i) {
        if (r > 0 && ends[r - 1] == sel[i]) ends[r - 1] = sel[i] + 1;
        else { starts[r] = sel[i]; ends[r] = sel[i] + 1; ++r; }
    }
    return r;
}

/* engine.py:145-154 attention_output over rows idx[0..k) (canonical logits).  out[d]. */
ORA_API void ora_attention(const double* q, const double* keys, const double* vals,
                           const int64_t* idx, int64_t k, int d, double* out) {
    for (int j = 0; j < d; ++j) out[j] = 0.0;
    if (k <= 0) return;
    double s = sqrt((double)d);
    double* w = (double*)malloc(sizeof(double) * (size_t)k);
    double mx = -INFINITY;
    for (int64_t i = 0; i < k; ++i) {
        w[i] = ora_dot(q, keys + idx[i] * (int64_t)d, d) / s;
        if (w[i] > mx) mx = w[i];
    }
    double sum = 0.0;
    for (int64_t i = 0; i < k; ++i) { w[i] = exp(w[i] - mx); sum += w[i]; }
    for (int64_t i = 0; i < k; ++i) {
        double wi = w[i] / sum;
        const double* v = vals + idx[i] * (int64_t)d;
        for (int j = 0; j < d; ++j) out[j] += wi * v[j];
    }
    free(w);
}

/* ------------------------------------------------------------------------------------ */
/* branch-and-bound partition (chunk_tree.py:171-379), restated                          */
/* ------------------------------------------------------------------------------------ */

enum { ST_CANDIDATE = 0, ST_IMPORTANT = 1, ST_DESERT = 2, ST_PAD = 3 };

typedef struct {
    int64_t start, end;
    double U, L;
    int state;
    int alive;
    double* mx; /* d doubles, NULL for pads */
    double* mn;
} node_t;

typedef struct {
    int64_t n, n_pad;
    int d;
    double* keys;   /* owned copy [n][d] */
    node_t* nodes;  /* every node ever created (arena) */
    int64_t n_nodes, cap_nodes;
    int64_t* leaves; /* indices of current leaves, sorted by start */
    int64_t n_leaves;
} ora_part_t;

static int64_t next_pow2_i64(int64_t n) {
    int64_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

static int64_t new_node(ora_part_t* P, int64_t start, int64_t end, int state) {
    if (P->n_nodes == P->cap_nodes) {
        P->cap_nodes = P->cap_nodes ? P->cap_nodes * 2 : 1024;
        P->nodes = (node_t*)realloc(P->nodes, sizeof(node_t) * (size_t)P->cap_nodes);
    }
    node_t* x = &P->nodes[P->n_nodes];
    x->start = start; x->end = end; x->U = NAN; x->L = NAN; x->state = state; x->alive = 1;
    x->mx = NULL; x->mn = NULL;
    if (state != ST_PAD) {
        x->mx = (double*)malloc(sizeof(double) * 2 * (size_t)P->d);
        x->mn = x->mx + P->d;
        int64_t e = end < P->n ? end : P->n;
        ora_abstract(P->keys, P->d, start, e, x->mx, x->mn);
    }
    return P->n_nodes++;
}

/* chunk_tree.py:171-210 build_partition(n, m, keys): m uniform leaves over next_pow2(n). */
ORA_API ora_part_t* ora_part_new(const double* keys, int64_t n, int d, int64_t m) {
    ora_part_t* P = (ora_part_t*)calloc(1, sizeof(ora_part_t));
    P->n = n; P->d = d; P->n_pad = next_pow2_i64(n);
    if (m < 1 || P->n_pad % m != 0) { free(P); return NULL; }
    P->keys = (double*)malloc(sizeof(double) * (size_t)(n * d));
    memcpy(P->keys, keys, sizeof(double) * (size_t)(n * d));
    int64_t size = P->n_pad / m;
    P->leaves = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
    for (int64_t s = 0; s < P->n_pad; s += size)
        P->leaves[P->n_leaves++] = new_node(P, s, s + size, s >= n ? ST_PAD : ST_CANDIDATE);
    return P;
}

ORA_API void ora_part_free(ora_part_t* P) {
    if (!P) return;
    for (int64_t i = 0; i < P->n_nodes; ++i) free(P->nodes[i].mx);
    free(P->nodes); free(P->leaves); free(P->keys); free(P);
}

/* The restated B&B evaluates bounds with the reference's own (numpy) arithmetic so that
 * its heap order, eval counts and leaf shapes reproduce kvtier's exactly. */
static void bound_node(ora_part_t* P, const double* q, node_t* x) {
    ora_bounds_ref(q, x->mx, x->mn, 1, P->d, &x->U, &x->L);
}

/* max-heap on (U desc, start asc) -- chunk_tree.py:270 key (-upper, start) */
typedef struct { int64_t* a; int64_t n; ora_part_t* P; } heap_t;

static int heap_less(heap_t* h, int64_t x, int64_t y) { /* x before y */
    node_t* a = &h->P->nodes[x];
    node_t* b = &h->P->nodes[y];
    if (a->U != b->U) return a->U > b->U;
    return a->start < b->start;
}
static void heap_push(heap_t* h, int64_t v) {
    int64_t i = h->n++;
    h->a[i] = v;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!heap_less(h, h->a[i], h->a[p])) break;
        int64_t t = h->a[i]; h->a[i] = h->a[p]; h->a[p] = t; i = p;
    }
}
static int64_t heap_pop(heap_t* h) {
    int64_t top = h->a[0];
    h->a[0] = h->a[--h->n];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, b = i;
        if (l < h->n && heap_less(h, h->a[l], h->a[b])) b = l;
        if (r < h->n && heap_less(h, h->a[r], h->a[b])) b = r;
        if (b == i) break;
        int64_t t = h->a[i]; h->a[i] = h->a[b]; h->a[b] = t; i = b;
    }
    return top;
}

static __thread ora_part_t* t_sort_P; /* qsort context, per thread */
static int cmp_leaf_start(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    int64_t sx = t_sort_P->nodes[x].start, sy = t_sort_P->nodes[y].start;
    return (sx > sy) - (sx < sy);
}

/* chunk_tree.py:233-338 select_top_k.  Writes confirmed tokens (confirmation order) to
 * out_tokens (capacity k), returns eval_count; -1 on bad k. */
ORA_API int64_t ora_part_select(ora_part_t* P, const double* q, int64_t k, int64_t* out_tokens) {
    if (k < 0 || k > P->n) return -1;
    int64_t evals = 0, conf = 0;
    /* live = real leaves */
    int64_t cap = P->n_leaves + 4 * P->n + 16;
    heap_t h; h.a = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap); h.n = 0; h.P = P;
    for (int64_t i = 0; i < P->n_leaves; ++i) {
        node_t* x = &P->nodes[P->leaves[i]];
        if (x->state == ST_PAD) continue;
        x->state = ST_CANDIDATE;
        bound_node(P, q, x);
        ++evals;
    }
    for (int64_t i = 0; i < P->n_leaves; ++i) {
        node_t* x = &P->nodes[P->leaves[i]];
        if (x->state != ST_PAD) heap_push(&h, P->leaves[i]);
    }
    while (conf < k && h.n > 0) {
        int64_t id = heap_pop(&h);
        node_t* x = &P->nodes[id];
        int64_t real_end = x->end < P->n ? x->end : P->n;
        int64_t real_size = real_end - x->start;
        int64_t budget = k - conf;
        if (real_size == 1) {
            x->state = ST_IMPORTANT;
            out_tokens[conf++] = x->start;
            continue;
        }
        double next_upper = h.n > 0 ? P->nodes[h.a[0]].U : -INFINITY;
        if (x->L > next_upper && real_size <= budget) {
            x->state = ST_IMPORTANT;
            for (int64_t t = x->start; t < real_end; ++t) out_tokens[conf++] = t;
            continue;
        }
        int64_t size = x->end - x->start;
        int64_t mid = x->start + size / 2;
        int64_t s0 = x->start, e1 = x->end;
        x->alive = 0;
        int64_t kids[2];
        (void)kids;
        int64_t los[2] = {s0, mid}, his[2] = {mid, e1};
        for (int c = 0; c < 2; ++c) {
            if (los[c] >= P->n) { kids[c] = new_node(P, los[c], his[c], ST_PAD); continue; }
            kids[c] = new_node(P, los[c], his[c], ST_CANDIDATE);
            x = NULL; /* nodes may have moved */
            bound_node(P, q, &P->nodes[kids[c]]);
            ++evals;
            if (h.n + 1 > cap) { cap *= 2; h.a = (int64_t*)realloc(h.a, sizeof(int64_t) * (size_t)cap); }
            heap_push(&h, kids[c]);
        }
    }
    for (int64_t i = 0; i < h.n; ++i) P->nodes[h.a[i]].state = ST_DESERT;
    free(h.a);
    /* rebuild leaves = alive nodes that are current leaves: every node created is a leaf
     * unless it was split (alive = 0).  Pads and merged-away nodes are tracked by alive. */
    int64_t nl = 0;
    for (int64_t i = 0; i < P->n_nodes; ++i) if (P->nodes[i].alive) ++nl;
    P->leaves = (int64_t*)realloc(P->leaves, sizeof(int64_t) * (size_t)(nl ? nl : 1));
    P->n_leaves = 0;
    for (int64_t i = 0; i < P->n_nodes; ++i) if (P->nodes[i].alive) P->leaves[P->n_leaves++] = i;
    t_sort_P = P;
    qsort(P->leaves, (size_t)P->n_leaves, sizeof(int64_t), cmp_leaf_start);
    return evals;
}

/* chunk_tree.py:344-379 merge_desert.  Returns merges done. */
ORA_API int64_t ora_part_merge(ora_part_t* P) {
    int64_t out = 0, merges = 0;
    for (int64_t i = 0; i < P->n_leaves; ++i) {
        int64_t id = P->leaves[i];
        node_t* x = &P->nodes[id];
        if (out > 0) {
            node_t* prev = &P->nodes[P->leaves[out - 1]];
            if (x->state == prev->state && (prev->state == ST_DESERT || prev->state == ST_PAD) &&
                prev->end == x->start) {
                int64_t pst = prev->start, xe = x->end;
                int st = prev->state;
                int64_t pid = P->leaves[out - 1];
                int64_t f = new_node(P, pst, xe, ST_PAD); /* no abstract from keys */
                node_t* fx = &P->nodes[f];
                prev = &P->nodes[pid]; x = &P->nodes[id];
                fx->state = st;
                if (st == ST_DESERT) {
                    fx->mx = (double*)malloc(sizeof(double) * 2 * (size_t)P->d);
                    fx->mn = fx->mx + P->d;
                    for (int j = 0; j < P->d; ++j) {
                        fx->mx[j] = prev->mx[j] > x->mx[j] ? prev->mx[j] : x->mx[j];
                        fx->mn[j] = prev->mn[j] < x->mn[j] ? prev->mn[j] : x->mn[j];
                    }
                }
                prev->alive = 0; x->alive = 0;
                P->leaves[out - 1] = f;
                ++merges;
                continue;
            }
        }
        P->leaves[out++] = id;
    }
    P->n_leaves = out;
    return merges;
}

ORA_API int64_t ora_part_n_leaves(const ora_part_t* P) { return P->n_leaves; }

/* leaf spans: starts/ends/states (capacity n_leaves) */
ORA_API void ora_part_leaves(const ora_part_t* P, int64_t* starts, int64_t* ends, int32_t* states) {
    for (int64_t i = 0; i < P->n_leaves; ++i) {
        const node_t* x = &P->nodes[P->leaves[i]];
        starts[i] = x->start; ends[i] = x->end; states[i] = x->state;
    }
}

/* abstract of leaf i (zeros if pad) */
ORA_API void ora_part_leaf_abstract(const ora_part_t* P, int64_t i, double* mx, double* mn) {
    const node_t* x = &P->nodes[P->leaves[i]];
    for (int j = 0; j < P->d; ++j) {
        mx[j] = x->mx ? x->mx[j] : 0.0;
        mn[j] = x->mx ? x->mn[j] : 0.0;
    }
}

/* ------------------------------------------------------------------------------------ */
/* multi-threaded lane-step baseline (bench.py cpu_baseline / --impl reference)          */
/* ------------------------------------------------------------------------------------ */

typedef struct {
    /* inputs */
    int64_t n; int d; int64_t m; int64_t k; int steps; int merge;
    const float* keys;    /* [lanes][n][d] */
    const float* vals;    /* [lanes][n][d] */
    const float* q;       /* [steps][lanes][d] */
    int64_t lanes;
    /* work split */
    int tid, nthreads;
    /* outputs */
    double* out;          /* [steps][lanes][d] attention outputs (may be NULL) */
    int64_t* evals;       /* [steps][lanes] */
    double timed_s;       /* per-thread time inside select+attention */
    double* lane_step_s;  /* [steps][lanes] time of each lane-step (NULL: not recorded) */
} bench_arg_t;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* bench_worker(void* p) {
    bench_arg_t* a = (bench_arg_t*)p;
    int d = a->d;
    int64_t n = a->n;
    double* k64 = (double*)malloc(sizeof(double) * (size_t)(n * d));
    double* v64 = (double*)malloc(sizeof(double) * (size_t)(n * d));
    double* q64 = (double*)malloc(sizeof(double) * (size_t)d);
    int64_t* tok = (int64_t*)malloc(sizeof(int64_t) * (size_t)(a->k > 0 ? a->k : 1));
    double* o = (double*)malloc(sizeof(double) * (size_t)d);
    a->timed_s = 0.0;
    for (int64_t lane = a->tid; lane < a->lanes; lane += a->nthreads) {
        const float* K = a->keys + lane * n * d;
        const float* V = a->vals + lane * n * d;
        for (int64_t i = 0; i < n * d; ++i) { k64[i] = K[i]; v64[i] = V[i]; }
        ora_part_t* P = ora_part_new(k64, n, d, a->m);           /* pre-built partition */
        for (int s = 0; s < a->steps; ++s) {
            const float* Q = a->q + ((int64_t)s * a->lanes + lane) * d;
            for (int j = 0; j < d; ++j) q64[j] = Q[j];
            double t0 = now_s();
            int64_t ev = ora_part_select(P, q64, a->k, tok);      /* chunk_tree.py:233 */
            qsort(tok, (size_t)a->k, sizeof(int64_t), cmp_i64);   /* engine.py:353 sorted */
            ora_attention(q64, k64, v64, tok, a->k, d, o);        /* engine.py:354 */
            if (a->merge) ora_part_merge(P);
            double dt = now_s() - t0;
            a->timed_s += dt;
            if (a->lane_step_s) a->lane_step_s[(int64_t)s * a->lanes + lane] = dt;
            if (a->evals) a->evals[(int64_t)s * a->lanes + lane] = ev;
            if (a->out) memcpy(a->out + ((int64_t)s * a->lanes + lane) * d, o, sizeof(double) * (size_t)d);
        }
        ora_part_free(P);
    }
    free(k64); free(v64); free(q64); free(tok); free(o);
    return NULL;
}

/* Runs `steps` decode steps over `lanes` independent lanes with a persistent partition per
 * lane (m uniform initial leaves), nthreads POSIX threads, lanes round-robin.  Returns the
 * wall-clock seconds of the whole timed phase (max over threads of their timed work is in
 * *max_thread_s).  Setup (widening, build_partition) is excluded, as in BASELINE.md sec. 3. */
ORA_API double ora_bench_lanes(int64_t lanes, int64_t n, int d, int64_t m, int64_t k, int steps,
                               int merge, const float* keys, const float* vals, const float* q,
                               int nthreads, double* out, int64_t* evals, double* max_thread_s,
                               double* sum_thread_s, double* lane_step_s) {
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    bench_arg_t* args = (bench_arg_t*)calloc((size_t)nthreads, sizeof(bench_arg_t));
    double t0 = now_s();
    for (int t = 0; t < nthreads; ++t) {
        bench_arg_t* a = &args[t];
        a->n = n; a->d = d; a->m = m; a->k = k; a->steps = steps; a->merge = merge;
        a->keys = keys; a->vals = vals; a->q = q; a->lanes = lanes;
        a->tid = t; a->nthreads = nthreads; a->out = out; a->evals = evals; a->lane_step_s = lane_step_s;
        pthread_create(&th[t], NULL, bench_worker, a);
    }
    double mx = 0.0, sum = 0.0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        if (args[t].timed_s > mx) mx = args[t].timed_s;
        sum += args[t].timed_s;
    }
    double wall = now_s() - t0;
    if (max_thread_s) *max_thread_s = mx;
    if (sum_thread_s) *sum_thread_s = sum;
    free(th); free(args);
    return wall;
}
