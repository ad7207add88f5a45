// score.cu -- K4 canonical float64 token logits (candidate tokens, or all tokens).
//
// Replaces importance.py:27-33 attention_logits (k.q / sqrt d) for the tokens the plan
// kept.  The pipeline keeps raw canonical dots (the 1/sqrt d scale does not change the
// order and is applied inside the softmax of K7); kvt_token_scores returns fl(dot)/fl(sqrt d).  A warp scores 8 tokens per step: each lane loads its 4-dim group of the 8 rows
// (8 independent 64/128-bit loads in flight per lane; a 128-dim bf16 row is one coalesced
// 256 B warp access), runs its f64 fma chains, and a reduce-scatter butterfly
// (tree_8tok: 9 f64 shuffles per 8 tokens instead of 40) yields the canonical dot of
// token (lane>>2) on every quad.  HBM-bound: n_cand*d*s_K read, n_cand*12 B written.
#include <type_traits>

#include "common.cuh"

namespace kvt {

constexpr int SCORE_THREADS = 256;

template <typename QT, typename T, int G, bool VEC, bool IMPLICIT>
__global__ void __launch_bounds__(SCORE_THREADS) score_kernel(
    const QT* __restrict__ q, const T* __restrict__ keys, int64_t lane_stride, int d,
    const int32_t* __restrict__ items, int64_t item_stride, const int32_t* __restrict__ n_items,
    int64_t n_implicit, double* __restrict__ out_score, int32_t* __restrict__ out_tok, int64_t out_stride,
    int scaled) {
    const int lane = threadIdx.x & 31;
    const int64_t li = blockIdx.y;
    double qr[G][4];
#pragma unroll
    for (int r = 0; r < G; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = 4 * (lane + 32 * r) + i;
            qr[r][i] = j < d ? (double)q[li * d + j] : 0.0;
        }
    const double sd = sqrt((double)d);
    const T* base = keys + li * lane_stride;
    const int64_t nit = IMPLICIT ? (n_implicit + 63) / 64 : (int64_t)n_items[li];
    const int32_t* itl = IMPLICIT ? nullptr : items + li * item_stride * 3;
    double* os = out_score + li * out_stride;
    int32_t* ot = out_tok ? out_tok + li * out_stride : nullptr;
    const int64_t wpb = SCORE_THREADS / 32;
    const int64_t nwarps = (int64_t)gridDim.x * wpb;

    for (int64_t it = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); it < nit; it += nwarps) {
        int64_t t0, cnt, pos0;
        if (IMPLICIT) {
            t0 = it * 64; cnt = kvt::imin(64, n_implicit - t0); pos0 = t0;
        } else {
            t0 = itl[it * 3 + 0]; cnt = itl[it * 3 + 1]; pos0 = itl[it * 3 + 2];
        }
        for (int64_t g8 = 0; g8 < cnt; g8 += 8) {
            double p[8];
            double v[8][G][4];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool ok = g8 + u < cnt;
                const T* row = base + (t0 + g8 + u) * (int64_t)d;
#pragma unroll
                for (int r = 0; r < G; ++r) {
                    const int g = lane + 32 * r;
                    if (ok && 4 * g < d) load_group<T, VEC>(row, g, d, v[u][r]);
                    else { v[u][r][0] = v[u][r][1] = v[u][r][2] = v[u][r][3] = 0.0; }
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                double acc = 0.0;
#pragma unroll
                for (int r = 0; r < G; ++r) {
                    const int g = lane + 32 * r;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (4 * g + i < d) acc = fma(qr[r][i], v[u][r][i], acc);
                }
                p[u] = acc;
            }
            const double dot = tree_8tok(p, lane);
            const int t = (lane >> 2) & 7;
            if ((lane & 3) == 0 && g8 + t < cnt) {
                os[pos0 + g8 + t] = scaled ? dot / sd : dot;
                if (ot) ot[pos0 + g8 + t] = (int32_t)(t0 + g8 + t);
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// TMA-pipelined variant (sm_100a): persistent CTAs walk the flattened (lane, item) list;
// one producer thread streams each 64-token item (a contiguous run of key rows) into a
// shared-memory ring with cp.async.bulk + mbarrier transaction counts, 8 consumer warps
// score 8 tokens each per item straight from shared memory.  Bytes in flight per CTA =
// stages x tile (64 KB for bf16 d=128), independent of the consumers' dependency chains.
// ------------------------------------------------------------------------------------------

constexpr int TS_CONSUMERS = 8;
constexpr int TS_THREADS = (TS_CONSUMERS + 1) * 32;

// AccT = double: canonical f64 dots (the exact definition); AccT = float: the fast f32
// estimate written to out32 (select3.cu brackets it with a rigorous error bound and
// re-scores the few tokens near the k-th value in f64, so the selected set stays exact).
template <typename QT, typename T, int G, bool IMPLICIT, typename AccT>
__global__ void __launch_bounds__(TS_THREADS, 3) score_tma_kernel(
    const QT* __restrict__ q, const unsigned char* __restrict__ keys, int64_t lane_stride_b, int row_b, int d,
    int n_lanes, const int32_t* __restrict__ items, int64_t item_stride, const int32_t* __restrict__ n_items,
    int64_t n_implicit, double* __restrict__ out_score, float* __restrict__ out32, int32_t* __restrict__ out_tok,
    int64_t out_stride, int stages, int tile_bytes, int scaled, int kvg) {
    pdl_entry();
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ long long scan_sh[33];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * tile_bytes);
    uint64_t* empty = full + stages;
    int4* meta = reinterpret_cast<int4*>(empty + stages);  // per stage: lane, t0, cnt, pos0
    int32_t* lane_off = reinterpret_cast<int32_t*>(meta + stages);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // prefix of per-lane item counts (the flattened work list)
    // one block scan: thread t owns a contiguous run of lanes (independent loads, one latency)
    long long carry = 0;
    {
        const int per = (n_lanes + TS_THREADS - 1) / TS_THREADS;
        const int a = min(n_lanes, tid * per), b = min(n_lanes, a + per);
        long long v = 0;
        for (int i = a; i < b; ++i) v += IMPLICIT ? (n_implicit + 63) / 64 : (long long)n_items[i];
        long long tot;
        long long run = block_excl_scan<long long>(v, scan_sh, tot);
        for (int i = a; i < b; ++i) {
            lane_off[i] = (int32_t)run;
            run += IMPLICIT ? (n_implicit + 63) / 64 : (long long)n_items[i];
        }
        carry = tot;
    }
    if (tid == 0) {
        lane_off[n_lanes] = (int32_t)carry;
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TS_CONSUMERS);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t total = lane_off[n_lanes];
    // contiguous block of the flattened list per CTA: the lane (and its query) changes rarely
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t g_begin = kvt::imin(total, (int64_t)blockIdx.x * per);
    const int64_t g_end = kvt::imin(total, g_begin + per);

    if (warp == TS_CONSUMERS) {  // ---- producer warp: lane 0 drives the bulk-copy engine ----
        // explicit item lists are read 32 items at a time (one load per lane, shuffled to
        // lane 0): one memory latency per batch instead of per item
        int cur = 0;
        {  // binary search: last lane with lane_off[lane] <= g_begin
            int lo = 0, hi = n_lanes - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (lane_off[mid] <= g_begin) lo = mid; else hi = mid - 1;
            }
            cur = lo;
        }
        int ps = 0, pr = 0;
        int64_t g = g_begin;
        while (g < g_end) {
            while (g >= lane_off[cur + 1]) ++cur;
            const int64_t it0 = g - lane_off[cur];
            const int nb = (int)kvt::imin((int64_t)32, kvt::imin((int64_t)lane_off[cur + 1] - g, g_end - g));
            int m0 = 0, m1 = 0, m2 = 0;
            if (!IMPLICIT && lane < nb) {
                const int32_t* m = items + ((int64_t)cur * item_stride + it0 + lane) * 3;
                m0 = m[0]; m1 = m[1]; m2 = m[2];
            }
            for (int j = 0; j < nb; ++j) {
                int64_t t0, cnt;
                int pos0;
                if (IMPLICIT) { t0 = (it0 + j) * 64; cnt = kvt::imin((int64_t)64, n_implicit - t0); pos0 = (int)t0; }
                else {
                    t0 = __shfl_sync(KVT_FULL, m0, j);
                    cnt = __shfl_sync(KVT_FULL, m1, j);
                    pos0 = __shfl_sync(KVT_FULL, m2, j);
                }
                const int s = ps;
                if (lane == 0) {
                    if (pr > 0) mbar_wait(&empty[s], (uint32_t)((pr - 1) & 1));
                    const uint32_t bytes = (uint32_t)(cnt * row_b);
                    meta[s] = make_int4(cur, (int)t0, (int)cnt, pos0);
                    mbar_arrive_expect_tx(&full[s], bytes);
                    bulk_g2s(smem + (size_t)s * tile_bytes, keys + (int64_t)(cur / kvg) * lane_stride_b + t0 * row_b, bytes,
                             &full[s]);
                }
                if (++ps == stages) { ps = 0; ++pr; }
            }
            g += nb;
        }
        return;
    }

    // ---- consumers: 8 warps x 8 tokens per 64-token item ----
    const double sd = sqrt((double)d);
    int cur = -1;
    AccT qr[G][4];
    float qg[std::is_same<T, I4>::value && sizeof(AccT) == 4 ? 32 : 1];  // INT4 fast path: a lane's 32-dim group of q
    int qcur_i4 = -1;
    int64_t i = 0;
    int cs = 0, cr = 0;
    for (int64_t g = g_begin; g < g_end; ++g, ++i) {
        const int s = cs;
        mbar_wait(&full[s], (uint32_t)(cr & 1));
        if (++cs == stages) { cs = 0; ++cr; }
        const int4 mt = meta[s];
        if (mt.x != cur) {
            cur = mt.x;
#pragma unroll
            for (int r = 0; r < G; ++r)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = 4 * (lane + 32 * r) + e;
                    qr[r][e] = j < d ? (AccT)q[(int64_t)cur * d + j] : (AccT)0;
                }
        }
        const int64_t t0 = mt.y, cnt = mt.z, pos0 = mt.w;
        const unsigned char* tile = smem + (size_t)s * tile_bytes;
        const int base_t = 8 * warp;
        if constexpr (std::is_same<T, I4>::value && sizeof(AccT) == 4) {
            // INT4 fast estimate: a token's record is read by LPT = d/32 lanes, one 32-dim group
            // each (16 B of codes + its (scale, min)), 4 independent fma chains of 8, then a
            // shuffle reduction over the token's lanes.  (Any order is fine for the f32
            // estimate: the plan's error bound covers <= chain_len(d) + 3 roundings.)
            constexpr int LPT = 4 * G;        // lanes per token (d = 128 G)
            constexpr int TPW = 32 / LPT;     // tokens per warp instruction
            const int grp = lane % LPT, sub = lane / LPT;
            if (cur != qcur_i4) {
                qcur_i4 = cur;
#pragma unroll
                for (int e = 0; e < 32; ++e) qg[e] = (float)q[(int64_t)cur * d + 32 * grp + e];
            }
#pragma unroll
            for (int rep = 0; rep < 8 / TPW; ++rep) {
                const int u = base_t + rep * TPW + sub;  // token within the item
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                if (u < cnt) {
                    const unsigned char* row = tile + (int64_t)u * row_b;
                    const uint4 cw = *reinterpret_cast<const uint4*>(row + 16 * grp);
                    const __half2 pr = *reinterpret_cast<const __half2*>(row + d / 2 + 4 * grp);
                    const float sc_ = __low2float(pr), mn = __high2float(pr);
                    const uint32_t wv[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
                    for (int wi = 0; wi < 4; ++wi) {
                        const uint32_t lo4 = wv[wi] & 0x0f0f0f0fu, hi4 = (wv[wi] >> 4) & 0x0f0f0f0fu;
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            // code -> float without I2F: one byte permute builds 0x4B0000cc = 2^23 + c
                            const float c0 = __uint_as_float(__byte_perm(0x4B000000u, lo4, 0x3004 + b)) - 8388608.0f;
                            const float c1 = __uint_as_float(__byte_perm(0x4B000000u, hi4, 0x3004 + b)) - 8388608.0f;
                            const int e = 8 * wi + 2 * b;
                            acc[wi] = fmaf(qg[e], __fmaf_rn(c0, sc_, mn), acc[wi]);
                            acc[wi] = fmaf(qg[e + 1], __fmaf_rn(c1, sc_, mn), acc[wi]);
                        }
                    }
                }
                float v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
                for (int off = 1; off < LPT; off <<= 1) v += __shfl_xor_sync(KVT_FULL, v, off);
                if (grp == 0 && u < cnt) {
                    out32[(int64_t)cur * out_stride + pos0 + u] = v;
                    if (out_tok) out_tok[(int64_t)cur * out_stride + pos0 + u] = (int32_t)(t0 + u);
                }
            }
        } else if (base_t < cnt) {
            AccT p[8];
            const unsigned char* rows = tile + (int64_t)base_t * row_b;
            if (base_t + 8 <= cnt && d == 128 * G) {
                // full group of 8 tokens, d a multiple of 128: no bounds checks
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    AccT acc = 0;
#pragma unroll
                    for (int r = 0; r < G; ++r) {
                        AccT v[4];
                        if constexpr (sizeof(AccT) == 8) RowLd<T>::load(rows + (int64_t)u * row_b, lane + 32 * r, d, v);
                        else RowLd<T>::loadf(rows + (int64_t)u * row_b, lane + 32 * r, d, v);
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc = fma(qr[r][e], v[e], acc);
                    }
                    p[u] = acc;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    AccT acc = 0;
                    if (base_t + u < cnt) {
                        const unsigned char* row = rows + (int64_t)u * row_b;
#pragma unroll
                        for (int r = 0; r < G; ++r) {
                            const int gg = lane + 32 * r;
                            if (4 * gg < d) {
                                AccT v[4];
                                if constexpr (sizeof(AccT) == 8) RowLd<T>::load(row, gg, d, v);
                                else RowLd<T>::loadf(row, gg, d, v);
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    if (4 * gg + e < d) acc = fma(qr[r][e], v[e], acc);
                            }
                        }
                    }
                    p[u] = acc;
                }
            }
            const AccT dot = tree_8tok<AccT>(p, lane);
            const int t = (lane >> 2) & 7;
            if ((lane & 3) == 0 && base_t + t < cnt) {
                if constexpr (sizeof(AccT) == 8) {
                    double* os = out_score + (int64_t)cur * out_stride;
                    os[pos0 + base_t + t] = scaled ? dot / sd : dot;
                } else {
                    out32[(int64_t)cur * out_stride + pos0 + base_t + t] = dot;
                }
                if (out_tok) out_tok[(int64_t)cur * out_stride + pos0 + base_t + t] = (int32_t)(t0 + base_t + t);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

}  // namespace kvt

using namespace kvt;

static inline int sgroups_for(int d) { return d <= 128 ? 1 : d <= 256 ? 2 : d <= 512 ? 4 : d <= 1024 ? 8 : 0; }

using kvt::sm_count;

// TMA path eligibility: whole-row bulk copies need 16 B aligned rows and lane bases.
// lane_stride is in elements (bytes for I4).
template <typename T>
static bool tma_ok(const void* keys, int64_t lane_stride, int d, int64_t n_lanes) {
    const int64_t row = RowLd<T>::row_bytes(d);
    const int64_t ls_b = std::is_same<T, I4>::value ? lane_stride : lane_stride * (int64_t)sizeof(T);
    return d % 4 == 0 && d <= 1024 && row % 16 == 0 && ((uintptr_t)keys % 16) == 0 && ls_b % 16 == 0 &&
           64 * row * 2 <= 160 * 1024 && n_lanes <= 16384;
}

template <typename QT, typename T, int G, bool IMPL, typename AccT = double>
static int launch_score_tma(const void* q, const void* keys, int64_t n_lanes, int64_t lane_stride, int d,
                            const int32_t* items, int64_t item_stride, const int32_t* n_items, int64_t n_impl,
                            double* os, int32_t* ot, int64_t ostr, int scaled, cudaStream_t st, float* os32 = nullptr) {
    const int row_b = RowLd<T>::row_bytes(d);
    const int64_t ls_b = std::is_same<T, I4>::value ? lane_stride : lane_stride * (int64_t)sizeof(T);
    const int tile = 64 * row_b;
    int stages = (int)kvt::imin(std::is_same<T, I4>::value ? 6 : 3, (150 * 1024) / tile);
    if (stages < 2) stages = 2;
    const size_t smem = (size_t)stages * tile + 32 * (size_t)stages + 4 * (size_t)(n_lanes + 1) + 16;
    KVT_PER_DEVICE(size_t, configured);
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(score_tma_kernel<QT, T, G, IMPL, AccT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        configured = 200 * 1024;
    }
    KVT_PER_DEVICE(int, per_sm);  // one per template instance and device
    if (!per_sm) per_sm = resident_per_sm(score_tma_kernel<QT, T, G, IMPL, AccT>, TS_THREADS, smem,
                                          smem <= 70 * 1024 ? 3 : (smem <= 110 * 1024 ? 2 : 1));
    const int grid = sm_count() * per_sm;
    launch_pdl(score_tma_kernel<QT, T, G, IMPL, AccT>, dim3(grid), dim3(TS_THREADS), smem, st, (const QT*)q, (const unsigned char*)keys, ls_b, row_b, d, (int)n_lanes, items, item_stride, n_items, n_impl,
        os, os32, ot, ostr, stages, tile, scaled, kv_group_current());
    return kvt_check_launch();
}

template <typename QT, typename T, int G, bool VEC, bool IMPL>
static void launch_score(const void* q, const void* keys, int64_t n_lanes, int64_t lane_stride, int d,
                         const int32_t* items, int64_t item_stride, const int32_t* n_items, int64_t n_impl,
                         double* os, int32_t* ot, int64_t ostr, int blocks, int scaled, cudaStream_t st) {
    dim3 grid(blocks, (unsigned)n_lanes);
    score_kernel<QT, T, G, VEC, IMPL><<<grid, SCORE_THREADS, 0, st>>>(
        (const QT*)q, (const T*)keys, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled);
}

template <typename QT, typename T, bool IMPL>
static int dispatch_score_t(const void* q, const void* keys, int64_t n_lanes, int64_t lane_stride, int d,
                            const int32_t* items, int64_t item_stride, const int32_t* n_items, int64_t n_impl,
                            double* os, int32_t* ot, int64_t ostr, int blocks, int scaled, cudaStream_t st) {
    if (tma_ok<T>(keys, lane_stride, d, n_lanes)) {
        switch (sgroups_for(d)) {
            case 1: return launch_score_tma<QT, T, 1, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled, st);
            case 2: return launch_score_tma<QT, T, 2, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled, st);
            default: break;
        }
    }
    const bool vec = ((uintptr_t)keys % (4 * sizeof(T)) == 0) && d % 4 == 0 && lane_stride % 4 == 0;
    switch (sgroups_for(d)) {
#define KVT_CASE(GG)                                                                                                  \
    case GG:                                                                                                          \
        if (vec) launch_score<QT, T, GG, true, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items,  \
                                                     n_impl, os, ot, ostr, blocks, scaled, st);                                \
        else launch_score<QT, T, GG, false, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items,     \
                                                  n_impl, os, ot, ostr, blocks, scaled, st);                                   \
        break;
        KVT_CASE(1) KVT_CASE(2) KVT_CASE(4) KVT_CASE(8)
#undef KVT_CASE
        default: return KVT_ERR_SHAPE;
    }
    return kvt_check_launch();
}

template <bool IMPL>
static int dispatch_score(const void* q, int q_dtype, const void* keys, int key_dtype, int64_t n_lanes,
                          int64_t lane_stride, int d, const int32_t* items, int64_t item_stride,
                          const int32_t* n_items, int64_t n_impl, double* os, int32_t* ot, int64_t ostr, int blocks,
                          int scaled, cudaStream_t st) {
#define KVT_K(QT, TT) \
    return dispatch_score_t<QT, TT, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, blocks, scaled, st)
    if (key_dtype == KVT_I4) {
        if ((d != 128 && d != 256) || !tma_ok<I4>(keys, lane_stride, d, n_lanes)) return KVT_ERR_SHAPE;
        if (q_dtype != KVT_F32 && q_dtype != KVT_F64) return KVT_ERR_DTYPE;
        if (d == 128)
            return q_dtype == KVT_F32
                ? launch_score_tma<float, I4, 1, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled, st)
                : launch_score_tma<double, I4, 1, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled, st);
        return q_dtype == KVT_F32
            ? launch_score_tma<float, I4, 2, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled, st)
            : launch_score_tma<double, I4, 2, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, scaled, st);
    }
    if (q_dtype == KVT_F32) {
        switch (key_dtype) {
            case KVT_F32: KVT_K(float, float);
            case KVT_F64: KVT_K(float, double);
            case KVT_BF16: KVT_K(float, __nv_bfloat16);
            case KVT_F16: KVT_K(float, __half);
        }
    } else if (q_dtype == KVT_F64) {
        switch (key_dtype) {
            case KVT_F32: KVT_K(double, float);
            case KVT_F64: KVT_K(double, double);
            case KVT_BF16: KVT_K(double, __nv_bfloat16);
            case KVT_F16: KVT_K(double, __half);
        }
    }
#undef KVT_K
    return KVT_ERR_DTYPE;
}

extern "C" int kvt_cand_score(const void* q, int q_dtype, const void* keys, int key_dtype, int64_t n_lanes,
                              int64_t lane_stride, int d, const int32_t* items, int64_t item_stride,
                              const int32_t* n_items, double* cand_score, int32_t* cand_tok, int64_t cand_stride,
                              int blocks_per_lane, void* stream) {
    if (!q || !keys || !items || !n_items || !cand_score || d < 1 || n_lanes < 0) return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    if (blocks_per_lane < 1) blocks_per_lane = 1;
    return dispatch_score<false>(q, q_dtype, keys, key_dtype, n_lanes, lane_stride, d, items, item_stride, n_items,
                                 0, cand_score, cand_tok, cand_stride, blocks_per_lane, 0, (cudaStream_t)stream);
}

extern "C" int kvt_token_scores(const void* q, int q_dtype, const void* keys, int key_dtype, int64_t n_lanes,
                                int64_t lane_stride, int64_t n, int d, double* out, int64_t out_stride, void* stream) {
    if (!q || !keys || !out || d < 1 || n < 0 || n_lanes < 0) return KVT_ERR_ARG;
    if (n_lanes == 0 || n == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    const int64_t items = (n + 63) / 64;
    int blocks = (int)kvt::imin((items + 7) / 8, kvt::imax(1, 2048 / n_lanes));
    if (blocks < 1) blocks = 1;
    return dispatch_score<true>(q, q_dtype, keys, key_dtype, n_lanes, lane_stride, d, nullptr, 0, nullptr, n, out,
                                nullptr, out_stride, blocks, 1, (cudaStream_t)stream);
}

// Fast f32 candidate scores (select3.cu pairs them with an error bound): float keys of
// every dtype except f64; requires the TMA path.
template <typename QT, typename T>
static int fast_t(const void* q, const void* keys, int64_t n_lanes, int64_t lane_stride, int d, const int32_t* items,
                  int64_t item_stride, const int32_t* n_items, float* cs32, int32_t* ct, int64_t cstride,
                  cudaStream_t st) {
    if (!tma_ok<T>(keys, lane_stride, d, n_lanes)) return KVT_ERR_SHAPE;
    if (d == 128)
        return launch_score_tma<QT, T, 1, false, float>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items,
                                                        0, nullptr, ct, cstride, 0, st, cs32);
    if (d == 256)
        return launch_score_tma<QT, T, 2, false, float>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items,
                                                        0, nullptr, ct, cstride, 0, st, cs32);
    return KVT_ERR_SHAPE;
}

extern "C" int kvt_cand_score_f32(const void* q, int q_dtype, const void* keys, int key_dtype, int64_t n_lanes,
                                  int64_t lane_stride, int d, const int32_t* items, int64_t item_stride,
                                  const int32_t* n_items, float* cs32, int32_t* ct, int64_t cstride, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!q || !keys || !items || !n_items || !cs32 || !ct || n_lanes < 0) return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
#define KVT_F(QT, TT) return fast_t<QT, TT>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, cs32, ct, cstride, st)
    if (q_dtype == KVT_F32) {
        switch (key_dtype) {
            case KVT_F32: KVT_F(float, float);
            case KVT_BF16: KVT_F(float, __nv_bfloat16);
            case KVT_F16: KVT_F(float, __half);
            case KVT_I4: KVT_F(float, I4);
        }
    } else if (q_dtype == KVT_F64) {
        switch (key_dtype) {
            case KVT_F32: KVT_F(double, float);
            case KVT_BF16: KVT_F(double, __nv_bfloat16);
            case KVT_F16: KVT_F(double, __half);
            case KVT_I4: KVT_F(double, I4);
        }
    }
#undef KVT_F
    return KVT_ERR_DTYPE;
}

bool kvt_fast_ok(int key_dtype, int d) { return key_dtype != KVT_F64 && (d == 128 || d == 256); }
