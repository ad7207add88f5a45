// plan.cu -- lower-bound threshold tau and candidate work items (pruning half of
// chunk_tree.py:233-338 select_top_k).
//
// tau* = max{x : sum of rows over leaves with L >= x is >= k}: at least k tokens score
// >= tau*, so the k-th best score is >= tau* and any leaf with U < tau* holds no top-k
// token (strictly below, ties included).  A 3-pass weighted radix select over the top 24
// bits of the orderable 64-bit keys of L (sign, exponent, 12 mantissa bits) finds the
// bucket of tau*; tau = the smallest value of that bucket <= tau* is used, which prunes
// within 2^-12 relative of the exact threshold and stays sound.  One CTA per lane; the
// keys are staged in shared memory once; histogram weights are row counts.
// Candidate leaves (U >= tau) are emitted in ascending token order as work items of
// <= 64 tokens: (tok_start, count, out_pos), out_pos = exclusive prefix of candidate rows.
// Runs of adjacent candidate leaves are merged: items start at a run's first token and at
// every multiple of 64 inside a run, and end at the next multiple of 64 or the run's end,
// so small leaves (C = 8 in the early layers) still give full 64-token items.
//
// GQA union mode (grp = g > 1, decode path): one CTA per KV lane.  tau_h is found for each of
// the g query lanes h of the group (their own bounds and k), and a leaf is a candidate when
// U_h >= tau_h for ANY h.  The union's items are emitted once per KV lane, so the scorer
// reads each candidate record once for all g heads; every query lane's candidate list is the
// union (a superset of its own candidates -- its exact top-k is unchanged, only eval_count
// grows).  The per-query-lane error record takes max U_h and max A over the union.
#include "common.cuh"

namespace kvt {

constexpr int PLAN_THREADS = 512;
constexpr int ITEM_TOKENS = 64;

__device__ __forceinline__ int64_t leaf_rows(const int32_t* ls, int64_t nl, int64_t c, int64_t n, int C) {
    if (ls) {
        const int64_t e = (c + 1 < nl) ? (int64_t)ls[c + 1] : n;
        return e - ls[c];
    }
    return min((int64_t)C, n - c * C);
}
__device__ __forceinline__ int64_t leaf_begin(const int32_t* ls, int64_t c, int C) {
    return ls ? (int64_t)ls[c] : c * C;
}

// GMAX 1: one query lane per CTA (512 threads, 3 CTAs per SM); GQA union over grp <= GMAX query
// lanes: one CTA per KV lane and SM (1024 threads for grp <= 4: the work is grp-fold per CTA)
template <int GMAX, int PT>
__global__ void __launch_bounds__(PT, GMAX == 1 ? 3 : 1) plan_kernel(
    int64_t n, int C, const int32_t* __restrict__ leaf_start, const int32_t* __restrict__ n_leaves,
    int64_t leaf_stride, const double* __restrict__ U, const double* __restrict__ L, int64_t bnd_stride,
    int64_t k, int32_t* __restrict__ items, int64_t item_stride, int32_t* __restrict__ n_items,
    int32_t* __restrict__ n_cand, int8_t* __restrict__ cand_leaf, int64_t* __restrict__ evals, int stage_cap,
    const double* __restrict__ A, double* __restrict__ err, double err_factor, int grp, int ua_cap) {
    pdl_entry();
    if (GMAX == 1) grp = 1;
    extern __shared__ __align__(16) unsigned char plan_smem[];
    uint64_t* kst = reinterpret_cast<uint64_t*>(plan_smem);  // staged keys (if they fit)
    int8_t* fl = reinterpret_cast<int8_t*>(plan_smem) + (size_t)stage_cap * 8;  // union flags (grp > 1)
    // 32-bit bins: a lane's rows sum to n <= 2^22 (checked at launch), and 32-bit shared atomics
    // are native adds where 64-bit ones are compare-and-swap loops that spin under contention
    __shared__ __align__(8) unsigned int hist[GMAX * 256];
    __shared__ unsigned long long sp_h[GMAX], sm_h[GMAX];
    __shared__ long long sr_h[GMAX];
    __shared__ long long scan_sh[33];
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ long long s_remaining;
    __shared__ int s_done;
    __shared__ double s_tau[GMAX];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t li = blockIdx.x;  // query lane, or KV lane when grp > 1
    const int64_t q0 = li * grp;    // first query lane of the group
    const int32_t* ls = leaf_start ? leaf_start + li * leaf_stride : nullptr;
    const int64_t nl = leaf_start ? (int64_t)n_leaves[li] : (n + C - 1) / C;
    const bool staged = nl <= stage_cap;
    // single head: U and A staged next to the keys when they fit, so the flag and compaction
    // passes read shared memory instead of paying two more dependent global round trips
    const bool ua = GMAX == 1 && staged && nl <= ua_cap;
    double* su = reinterpret_cast<double*>(plan_smem + (size_t)stage_cap * 8);
    double* sa = su + ua_cap;
    // GQA: all heads' keys staged at once -> one histogram pass per digit serves every head
    const bool conc = GMAX > 1 && grp > 1 && (int64_t)grp * nl <= stage_cap;

    if (conc) {
        const int nl32 = (int)nl, tot = grp * nl32;
        for (int e = tid; e < tot; e += PT) {
            const int h = e / nl32;
            kst[e] = ord_key(L[(q0 + h) * bnd_stride + (e - h * nl32)]);
        }
        if (tid < GMAX) { sp_h[tid] = 0; sm_h[tid] = 0; sr_h[tid] = k; }
        __syncthreads();
        for (int shift = 56; shift >= 40 && k > 0; shift -= 8) {
            for (int i = tid; i < GMAX * 256; i += PT) hist[i] = 0;
            __syncthreads();
            for (int base = 0; base < tot; base += PT) {
                const int e = base + tid;
                int bin = GMAX * 256;
                unsigned long long w = 0;
                if (e < tot) {
                    const int h = e / nl32;
                    const int64_t c = e - h * nl32;
                    const uint64_t key = kst[e];
                    if ((key & sm_h[h]) == sp_h[h]) {
                        bin = h * 256 + (int)((key >> shift) & 0xff);
                        w = (unsigned long long)leaf_rows(ls, nl, c, n, C);
                    }
                }
                const unsigned peers = __match_any_sync(KVT_FULL, bin);
                const unsigned sum = __reduce_add_sync(peers, (unsigned)w);
                if (bin < GMAX * 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], sum);
            }
            __syncthreads();
            const int wh = tid >> 5;
            if (wh < grp) {  // warp h: the digit of head h (same scan as below)
                const unsigned int* hh = hist + wh * 256;
                unsigned long long loc = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) loc += hh[255 - 8 * lane - i];
                const unsigned long long inc = warp_incl_scan(loc, lane);
                const unsigned long long exc = inc - loc;
                const unsigned long long rem = (unsigned long long)sr_h[wh];
                const unsigned long long prefix = sp_h[wh], mask = sm_h[wh];
                __syncwarp();
                if (exc < rem && rem <= inc) {
                    unsigned long long run = exc;
                    for (int i = 0; i < 8; ++i) {
                        const int b = 255 - 8 * lane - i;
                        if (run + hh[b] >= rem) {
                            sp_h[wh] = prefix | ((unsigned long long)b << shift);
                            sm_h[wh] = mask | (0xffull << shift);
                            sr_h[wh] = (long long)(rem - run);
                            break;
                        }
                        run += hh[b];
                    }
                }
            }
            __syncthreads();
        }
        if (tid < grp) s_tau[tid] = (k <= 0) ? INFINITY : key_to_double(sp_h[tid]);
        __syncthreads();
        for (int64_t c = tid; c < nl; c += PT) {
            int8_t f = 0;
            for (int h = 0; h < grp; ++h) f |= U[(q0 + h) * bnd_stride + c] >= s_tau[h] ? 1 : 0;
            fl[c] = f;
        }
        __syncthreads();
    }

    for (int h = 0; h < grp && !conc; ++h) {
        const double* Ll = L + (q0 + h) * bnd_stride;
        if (ua) {
            const double* Uh = U + (q0 + h) * bnd_stride;
            const double* Ah = A ? A + (q0 + h) * bnd_stride : nullptr;
            for (int64_t c = tid; c < nl; c += PT) {
                const double lv = Ll[c], uv = Uh[c], av = Ah ? Ah[c] : 0.0;
                kst[c] = ord_key(lv);
                su[c] = uv;
                sa[c] = av;
            }
        } else if (staged) {
            for (int64_t c = tid; c < nl; c += PT) kst[c] = ord_key(Ll[c]);
        }
        if (tid == 0) { s_prefix = 0; s_mask = 0; s_remaining = k; s_done = (k <= 0); }
        __syncthreads();

        // ---- weighted radix select on the top 24 key bits ----
        for (int shift = 56; shift >= 40 && !s_done; shift -= 8) {
            for (int i = tid; i < 256; i += PT) hist[i] = 0;
            __syncthreads();
            const unsigned long long prefix = s_prefix, mask = s_mask;
            for (int64_t base = 0; base < nl; base += PT) {
                const int64_t c = base + tid;
                int digit = 256;
                unsigned long long w = 0;
                if (c < nl) {
                    const uint64_t key = staged ? kst[c] : ord_key(Ll[c]);
                    if ((key & mask) == prefix) {
                        digit = (int)((key >> shift) & 0xff);
                        w = (unsigned long long)leaf_rows(ls, nl, c, n, C);
                    }
                }
                // warp-aggregated weighted histogram: leaves are disjoint, so 32 row counts sum to <= n
                const unsigned peers = __match_any_sync(KVT_FULL, digit);
                const unsigned sum = __reduce_add_sync(peers, (unsigned)w);
                if (digit < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[digit], sum);
            }
            __syncthreads();
            if (tid < 32) {
                // lane covers bins 255-8*lane .. 248-8*lane (descending)
                unsigned long long loc = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) loc += hist[255 - 8 * lane - i];
                unsigned long long inc = warp_incl_scan(loc, lane);
                const unsigned long long exc = inc - loc;
                const unsigned long long rem = (unsigned long long)s_remaining;
                __syncwarp();  // all lanes have read s_remaining before one lane rewrites it
                const bool mine = exc < rem && rem <= inc;
                if (mine) {
                    unsigned long long run = exc;
                    for (int i = 0; i < 8; ++i) {
                        const int b = 255 - 8 * lane - i;
                        if (run + hist[b] >= rem) {
                            s_prefix = prefix | ((unsigned long long)b << shift);
                            s_mask = mask | (0xffull << shift);
                            s_remaining = (long long)(rem - run);
                            break;
                        }
                        run += hist[b];
                    }
                }
            }
            __syncthreads();
        }
        const double tau_h = (k <= 0) ? INFINITY : key_to_double(s_prefix);
        if (tid == 0) s_tau[h] = tau_h;
        if (grp > 1 && staged) {  // union flags: OR over the group's heads
            const double* Uh = U + (q0 + h) * bnd_stride;
            for (int64_t c = tid; c < nl; c += PT) {
                const int8_t f = Uh[c] >= tau_h ? 1 : 0;
                fl[c] = h == 0 ? f : (int8_t)(fl[c] | f);
            }
        }
        __syncthreads();
    }
    const double tau = s_tau[0];
    const double* Ul = U + q0 * bnd_stride;

    // ---- candidate flags (single head: staged over the keys, which are no longer needed) ----
    int8_t* fl1 = reinterpret_cast<int8_t*>(plan_smem);
    if (grp == 1 && staged)
        for (int64_t c = tid; c < nl; c += PT) fl1[c] = (ua ? su[c] : Ul[c]) >= tau ? 1 : 0;
    __syncthreads();
    auto is_cand = [&](int64_t c) -> bool {
        if (staged) return (grp == 1 ? fl1[c] : fl[c]) != 0;
        for (int h = 0; h < grp; ++h)
            if (U[(q0 + h) * bnd_stride + c] >= s_tau[h]) return true;
        return false;
    };

    // ---- candidate compaction -> items (+ max A / max U over candidates, per query lane) ----
    long long carry_items = 0, carry_tok = 0;
    double amax_c[GMAX], umax_c[GMAX];
#pragma unroll
    for (int h = 0; h < GMAX; ++h) { amax_c[h] = 0.0; umax_c[h] = -INFINITY; }
    for (int64_t base = 0; base < nl; base += PT) {
        const int64_t c = base + tid;
        long long it = 0, tk = 0;
        int64_t rows = 0, s = 0, first = 0;
        bool cand = false;
        if (c < nl) {
            rows = leaf_rows(ls, nl, c, n, C);
            s = leaf_begin(ls, c, C);
            cand = is_cand(c);
            if (cand) {
                tk = rows;
                const bool run_start = c == 0 || !is_cand(c - 1);
                first = (run_start || s % ITEM_TOKENS == 0) ? s : (s / ITEM_TOKENS + 1) * ITEM_TOKENS;
                const int64_t e = s + rows;
                it = first < e ? 1 + ((e - 1) / ITEM_TOKENS - first / ITEM_TOKENS) : 0;
#pragma unroll
                for (int h = 0; h < GMAX; ++h) {
                    if (h < grp) {
                        if (A) amax_c[h] = fmax(amax_c[h], ua ? sa[c] : A[(q0 + h) * bnd_stride + c]);
                        umax_c[h] = fmax(umax_c[h], ua ? su[c] : U[(q0 + h) * bnd_stride + c]);
                    }
                }
            }
            if (cand_leaf) cand_leaf[li * leaf_stride + c] = cand ? 1 : 0;
        }
        // one scan of (items << 40 | tokens): items < 2^23 and tokens < 2^40 per lane
        long long tot_pk;
        const long long ex_pk = block_excl_scan<long long>((it << 40) | tk, scan_sh, tot_pk);
        const long long ex_it = ex_pk >> 40, ex_tk = ex_pk & ((1LL << 40) - 1);
        const long long tot_it = tot_pk >> 40, tot_tk = tot_pk & ((1LL << 40) - 1);
        if (it > 0) {
            const int64_t e = s + rows;
            int32_t* out = items + li * item_stride * 3;
            int64_t t = first;
            for (long long j = 0; j < it; ++j) {
                const int64_t nxt = (t / ITEM_TOKENS + 1) * ITEM_TOKENS;
                int64_t end = nxt;
                if (nxt > e) {  // the item may run on into the following candidate leaves
                    int64_t cc = c + 1, ce = e;
                    while (ce < nxt && cc < nl && is_cand(cc)) { ce += leaf_rows(ls, nl, cc, n, C); ++cc; }
                    end = ce < nxt ? ce : nxt;
                }
                const int64_t pos = carry_items + ex_it + j;
                out[pos * 3 + 0] = (int32_t)t;
                out[pos * 3 + 1] = (int32_t)(end - t);
                out[pos * 3 + 2] = (int32_t)(carry_tok + ex_tk + (t - s));
                t = nxt;
            }
        }
        carry_items += tot_it;
        carry_tok += tot_tk;
    }
    if (err) {
        // err record per query lane: [bound on |f32 estimate - canonical dot|, tau, max U over candidates, 0]
        __syncthreads();
        double* red = reinterpret_cast<double*>(hist);  // 64 x 8 B: [amax | umax] x <= 32 warps
        for (int h = 0; h < grp; ++h) {
            double am = 0.0, um = -INFINITY;
#pragma unroll
            for (int x = 0; x < GMAX; ++x)
                if (x == h) { am = amax_c[x]; um = umax_c[x]; }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                am = fmax(am, __shfl_xor_sync(KVT_FULL, am, off));
                um = fmax(um, __shfl_xor_sync(KVT_FULL, um, off));
            }
            if (lane == 0) { red[tid >> 5] = am; red[32 + (tid >> 5)] = um; }
            __syncthreads();
            if (tid == 0) {
                double m = 0.0, umx = -INFINITY;
                for (int w = 0; w < PT / 32; ++w) { m = fmax(m, red[w]); umx = fmax(umx, red[32 + w]); }
                err[(q0 + h) * 4 + 0] = m * err_factor;
                err[(q0 + h) * 4 + 1] = s_tau[h];
                err[(q0 + h) * 4 + 2] = umx;
                err[(q0 + h) * 4 + 3] = 0.0;
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        n_items[li] = (int32_t)carry_items;
        for (int h = 0; h < grp; ++h) {
            n_cand[q0 + h] = (int32_t)carry_tok;
            if (evals) evals[q0 + h] = (int64_t)nl + carry_tok;
        }
    }
}

}  // namespace kvt

using namespace kvt;

// Rigorous bound on |f32 estimate - canonical f64 dot| relative to A = sum |q_j| |k_j|:
// the f32 path (q rounded to f32: 1 unit; fma chain + tree: n = chain_len(d) units of
// 2^-24, gamma_n) plus the canonical f64 path's own error (n units of 2^-53), with slack.
// The f32 paths use at most chain_len(d) + 3 roundings per term: the row layout (4 dims per
// lane, tree of 5) or the INT4 layout (32 dims per lane in 4 chains of 8, 2 pairwise adds,
// <= 3 shuffle levels).
static double f32_err_factor(int d) {
    const int n = chain_len(d) + 3;
    return ((double)(n + 2) * 0x1p-24) * (1.0 + 0x1p-10) + (double)(n + 2) * 0x1p-52;
}

extern "C" int kvt_select_plan(int64_t n_lanes, int64_t n, int C, const int32_t* leaf_start, const int32_t* n_leaves,
                               int64_t leaf_stride, const double* U, const double* L, int64_t bnd_stride, int64_t k,
                               int32_t* items, int64_t item_stride, int32_t* n_items, int32_t* n_cand,
                               int8_t* cand_leaf, int64_t* evals, void* stream) {
    return kvt_select_plan2(n_lanes, n, C, leaf_start, n_leaves, leaf_stride, U, L, bnd_stride, k, items,
                               item_stride, n_items, n_cand, cand_leaf, evals, nullptr, nullptr, 0, stream);
}

extern "C" int kvt_select_plan2(int64_t n_lanes, int64_t n, int C, const int32_t* leaf_start, const int32_t* n_leaves,
                        int64_t leaf_stride, const double* U, const double* L, int64_t bnd_stride, int64_t k,
                        int32_t* items, int64_t item_stride, int32_t* n_items, int32_t* n_cand, int8_t* cand_leaf,
                        int64_t* evals, const double* A, double* err, int d, void* stream) {
    return kvt_select_plan_group(n_lanes, n, C, leaf_start, n_leaves, leaf_stride, U, L, bnd_stride, k, items,
                                 item_stride, n_items, n_cand, cand_leaf, evals, A, err, d, 1, stream);
}

extern "C" int kvt_select_plan_group(int64_t n_lanes, int64_t n, int C, const int32_t* leaf_start,
                                     const int32_t* n_leaves, int64_t leaf_stride, const double* U, const double* L,
                                     int64_t bnd_stride, int64_t k, int32_t* items, int64_t item_stride,
                                     int32_t* n_items, int32_t* n_cand, int8_t* cand_leaf, int64_t* evals,
                                     const double* A, double* err, int d, int grp, void* stream) {
    if (grp < 1 || grp > 8 || n_lanes % grp || (grp > 1 && leaf_start)) return KVT_ERR_ARG;
    if (!U || !L || !items || !n_items || !n_cand || n_lanes < 0 || n < 0) return KVT_ERR_ARG;
    if (!leaf_start && C < 1) return KVT_ERR_ARG;
    if (k < 0 || k > n) return KVT_ERR_K;
    if (n > (1LL << 22)) return KVT_ERR_SHAPE;  // packed (items, tokens) scan: <= 4M tokens per lane
    if (n_lanes == 0) return KVT_OK;
    if (n_lanes > 2147483647LL) return KVT_ERR_ARG;
    KVT_PER_DEVICE(bool, configured);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(plan_kernel<1, PLAN_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(plan_kernel<1, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(plan_kernel<4, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 9);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(plan_kernel<8, PLAN_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 9);
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        configured = true;
    }
    const int64_t max_leaves = leaf_start ? leaf_stride : (n + C - 1) / C;
    const int cap = (int)kvt::imin(max_leaves * grp, 16384);
    const int ua_cap = grp == 1 && max_leaves <= 4096 ? (int)max_leaves : 0;  // U, A staging (16 B per leaf)
    const size_t smem = (size_t)cap * (grp > 1 ? 9 : 8) + (size_t)ua_cap * 16;
    // fewer lanes than SMs (small batch): one CTA per SM anyway, so use 1024 threads
    const bool wide1 = grp == 1 && n_lanes < (int64_t)kvt::sm_count();
    auto kern = grp == 1 ? (wide1 ? plan_kernel<1, 1024> : plan_kernel<1, PLAN_THREADS>)
                         : grp <= 4 ? plan_kernel<4, 1024> : plan_kernel<8, PLAN_THREADS>;
    const int pt = grp > 4 || (grp == 1 && !wide1) ? PLAN_THREADS : 1024;
    launch_pdl(kern, dim3((unsigned)(n_lanes / grp)), dim3(pt), smem, (cudaStream_t)stream, n, C,
               leaf_start, n_leaves, leaf_stride, U, L, bnd_stride, k, items, item_stride, n_items, n_cand, cand_leaf,
               evals, cap, A, err, f32_err_factor(d), grp, ua_cap);
    return kvt_check_launch();
}
