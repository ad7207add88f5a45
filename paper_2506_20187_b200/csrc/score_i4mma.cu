// score_i4mma.cu -- K4 fast estimates for INT4 key records on the integer tensor cores.
//
// The candidate logits of importance.py:27-33 over INT4 records (quant.cu) are estimated as
//     est(t) = sum_g [ s_g(t) * inner_g(t) + m_g(t) * Qt_g ],   inner_g = sum_{j in g} c_j(t) qt_j
// with c_j the 4-bit codes, (s_g, m_g) the group's fp16 (scale, min) and qt a decomposition of
// the query into P = 4 signed 8-bit digits on power-of-two scales,
//     qt_j = sum_p s_p qi_{p,j},   s_p = s_0 2^-7p,   |qi| <= 127.
// inner_g is then an exact integer combination: one m16n8k32 s8 MMA per (8 dims of each of 4
// groups) x 16 tokens sums c_j qi_{p,j} exactly in int32, the record's nibbles become MMA
// operands with one mask (lo) or shift+mask (hi) per 4 codes -- the K order is permuted to the
// nibble order and the query digits are laid out to match (kvt_i4_qprep).  The epilogue is a
// few f32 fmas per (token, group): the MMA partials D_p (|D_p| < 2^16) and the power-of-two
// digit scales make every product exact, so est(t) carries <= 10 f32 roundings per group
// (<= 3 in inner_g -- 1 as evaluated, s_1 (128 D_0 + D_1) + s_3 (128 D_2 + D_3) --, the
// m_g Qt_g product and its fma, the r-accumulation, the group tree).  A
// rigorous per-token bound
//     |est32(t) - canonical f64 dot(t)| <= e(t) = 1.001 [u |est32(t)| + sum_g (15|s_g| + |m_g|) W_g]
// (u = 2^-24) covers the final rounding, the epilogue roundings (11 u qd_g, qd_g = sum over the
// group of sum_p s_p |qi_p|, which bounds |inner_g| / 15 and |Qt_g|, incl. Qt_g's own f32
// rounding), the digit residual q - qt, the canonical dot's own f64 rounding and the fp32
// rounding of the dequantised element the canonical dot sees; W_g per lane and group comes
// from kvt_i4_qprep.  One head per KV lane (QG = 1) takes the per-lane
//     E = 1.001 [u max_t |est32(t)| + sum_g max_t (15|s_g| + |m_g|) W_g] >= max_t e(t)
// (no per-token reductions; K5 time unchanged at config 3); GQA keeps max_t e(t) (the
// per-row maxima cost it spills).
// The per-lane bound is atomically max-ed into err[4 lane + 3], where
// the band select (select3) takes it as E: the band is then a few ulps wide and the
// selected set stays the exact canonical top-k.
//
// Dataflow: the persistent TMA ring of score.cu (one producer thread issuing cp.async.bulk
// of 64-token items, plus the lane's digit block on a lane change), 4 consumer warps, warp w
// owning tokens 16w..16w+15 of the item.  Per 16 tokens and 128 dims a warp issues 2 LDS.128
// of codes, 8 MMAs and ~40 f32 ops -- a few instructions per token instead of the ~4 per dim
// of CUDA-core dequantisation.
//
// GQA union mode (QG = group size > 1, kvt_select_plan_group items): items are per KV lane,
// so each candidate record is read from HBM once for all QG query lanes of the group, and
// the heads fill the MMA's N dimension instead of zero padding.  The K order of one MMA is
// then the 32 dims of ONE group (thread tig holds word tig of the group's 16 code bytes),
// and column n = 2h + (p & 1) carries digit p of head h (parts 0,1 in the first MMA, 2,3 in
// the second): per 16 tokens and 128 dims still 8 MMAs, now for 4 heads, and thread tig
// owns head tig's partials of every group -- the epilogue needs no shuffles.  Heads 4..7
// (QG = 8) take a second pass with their digits reloaded (L1).  Token ids are written once,
// in the group's first query-lane row.
#include <cfloat>
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace kvt {

constexpr int QM_CONSUMERS = 4;
constexpr int QM_THREADS = (QM_CONSUMERS + 1) * 32;
#ifndef KVT_QM_STAGES
#define KVT_QM_STAGES 3
#endif
#ifndef KVT_QM_MINB
#define KVT_QM_MINB 6
#endif
constexpr int QM_STAGES = KVT_QM_STAGES;  // build-time knobs for A/B runs (stages x CTAs per SM)
constexpr int QM_ROWS = 128;  // rows per stage: up to two contiguous 64-token plan items

__host__ __device__ __forceinline__ int qprep_bytes(int d) { return (d / 32) * 144 + 16; }

// ---- query digits: one warp per lane ---------------------------------------------------------
// Block layout per lane: [G][4 parts][4 i][b0, b1] (G*128 B) | [G](Qt_g f32, W_g f32, 0, 0) |
// s_0..s_3 f32.
// b0 byte j = qi_p[32g + 8i + 2j], b1 byte j = qi_p[32g + 8i + 2j + 1] (the nibble order).
template <typename QT>
__global__ void qprep_kernel(const QT* __restrict__ q, int64_t n_lanes, int d, unsigned char* __restrict__ out) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const int64_t li = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (li >= n_lanes) return;
    const int G = d / 32;
    const QT* ql = q + li * d;
    unsigned char* blk = out + li * (int64_t)qprep_bytes(d);
    double mx = 0.0;
    for (int g = 0; g < G; ++g) mx = fmax(mx, fabs((double)ql[32 * g + lane]));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(KVT_FULL, mx, off));
    double s0 = 1.0;
    if (mx > 0.0) {
        int e;
        frexp(mx / 127.0, &e);
        s0 = ldexp(1.0, e);
    }
    // canonical dot rounding depth n = 4 ceil(d / 128) + 5 (plan.cu, oracle.bounds)
    const double n_can = 4.0 * ((d + 127) / 128) + 5.0;
    const double u = 0x1p-24;
    unsigned char* cst = blk + G * 128;
    for (int g = 0; g < G; ++g) {
        const int e = lane;  // element within the group
        const double qv = (double)ql[32 * g + e];
        double r = qv, qt = 0.0, qd = 0.0;
        const int off = 8 * (e >> 3) + 4 * (e & 1) + ((e & 7) >> 1);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const double sp = ldexp(s0, -7 * p);
            double di = rint(r / sp);
            di = fmin(127.0, fmax(-127.0, di));
            blk[g * 128 + p * 32 + off] = (unsigned char)(signed char)(int)di;
            qt += di * sp;  // exact: few significant bits
            qd += fabs(di) * sp;
            r = qv - qt;
        }
        double qabs = fabs(qv), r1 = fabs(r), qts = qt;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            qabs += __shfl_xor_sync(KVT_FULL, qabs, o);
            r1 += __shfl_xor_sync(KVT_FULL, r1, o);
            qd += __shfl_xor_sync(KVT_FULL, qd, o);
            qts += __shfl_xor_sync(KVT_FULL, qts, o);  // exact: multiples of s_3, < 2^40 s_3
        }
        if (lane == 0) {
            // W_g: canonical f64 ((2n+4) 2^-53) and the dequantised element's f32 rounding (u)
            // on sum|q|, the digit residual, and 11 u on qd for the f32 epilogue (module
            // header).  1% slack for the f64 evaluation here; rounded up to f32.
            const double w = 1.01 * (qabs * ((2.0 * n_can + 4.0) * 0x1p-53 + u) + r1 * (1.0 + 0x1p-40) +
                                     11.0 * u * (1.0 + 0x1p-10) * qd) + DBL_MIN;
            float fw = (float)w;
            if ((double)fw < w) fw = nextafterf(fw, INFINITY);
            float* c4 = reinterpret_cast<float*>(cst + 16 * g);
            c4[0] = (float)qts;
            c4[1] = fw;
            c4[2] = 0.f;
            c4[3] = 0.f;
        }
    }
    if (lane < 4) reinterpret_cast<float*>(blk + G * 144)[lane] = (float)ldexp(s0, -7 * lane);
}

__device__ __forceinline__ void mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---- the scoring kernel --------------------------------------------------------------------
template <int R, int QG>  // R = d / 128 rounds of 4 groups; QG = query lanes per item row (GQA union)
__global__ void __launch_bounds__(QM_THREADS, KVT_QM_MINB) score_i4mma_kernel(
    const unsigned char* __restrict__ keys, int64_t lane_stride_b, int n_lanes, const int32_t* __restrict__ items,
    int64_t item_stride, const int32_t* __restrict__ n_items, const unsigned char* __restrict__ qprep,
    float* __restrict__ out32, int32_t* __restrict__ out_tok, int64_t out_stride, double* __restrict__ err, int kvg) {
    pdl_entry();
    constexpr int d = 128 * R;
    constexpr int G = 4 * R;
    constexpr int row_b = d / 2 + G * 4;
    constexpr int tile_b = QM_ROWS * row_b;
    constexpr int qb = G * 144 + 16;
    constexpr int stage_b = (tile_b + QG * qb + 15) / 16 * 16;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[QM_STAGES], empty[QM_STAGES];
    __shared__ int4 meta[QM_STAGES];
    __shared__ long long scan_sh[33];
    __shared__ long long start_info[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // flattened item list: find the first lane of this CTA's contiguous range (one block scan)
    long long total;
    {
        const int per = (n_lanes + QM_THREADS - 1) / QM_THREADS;
        const int a = min(n_lanes, tid * per), b = min(n_lanes, a + per);
        long long v = 0;
        for (int i = a; i < b; ++i) v += n_items[i];
        long long run = block_excl_scan<long long>(v, scan_sh, total);
        const long long per_cta = (total + gridDim.x - 1) / gridDim.x;
        const long long g0 = min(total, (long long)blockIdx.x * per_cta);
        for (int i = a; i < b; ++i) {
            const long long c = n_items[i];
            if (c > 0 && g0 >= run && g0 < run + c) { start_info[0] = i; start_info[1] = g0 - run; }
            run += c;
        }
        if (tid == 0) {
            for (int s = 0; s < QM_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], QM_CONSUMERS); }
            fence_mbar_init();
        }
    }
    __syncthreads();
    const long long per_cta = (total + gridDim.x - 1) / gridDim.x;
    const long long g_begin = min(total, (long long)blockIdx.x * per_cta);
    const long long g_end = min(total, g_begin + per_cta);
    const long long n_my = g_end - g_begin;

    if (warp == QM_CONSUMERS) {  // ---- producer warp: lane 0 drives the bulk-copy engine ----
        // Item metadata is fetched 32 items at a time (one coalesced load per lane, handed to
        // lane 0 by shuffles), so the issue loop pays one memory latency per batch, not per item.
        // Consecutive items of a lane that continue each other (tokens and output positions)
        // are merged into one stage of up to QM_ROWS rows: one bulk copy, two MMA tiles per warp.
        // A final stage with cnt = -1 tells the consumers to stop.
        int ps = 0, pr = 0;
        if (n_my > 0) {
            int cur = (int)start_info[0];
            long long it = start_info[1];
            long long cnt_cur = n_items[cur];
            long long cnt_next = cur + 1 < n_lanes ? n_items[cur + 1] : 0;
            int prev = -1;
            long long g = 0;
            while (g < n_my) {
                while (it >= cnt_cur) {
                    ++cur;
                    it = 0;
                    cnt_cur = cnt_next;
                    cnt_next = cur + 1 < n_lanes ? n_items[cur + 1] : 0;
                }
                const int nb = (int)min(32LL, min(cnt_cur - it, n_my - g));
                int m0 = 0, m1 = 0, m2 = 0;
                if (lane < nb) {
                    const int32_t* m = items + ((int64_t)cur * item_stride + it + lane) * 3;
                    m0 = m[0]; m1 = m[1]; m2 = m[2];
                }
                for (int j = 0; j < nb; ++j) {
                    const int t0 = __shfl_sync(KVT_FULL, m0, j);
                    int cnt = __shfl_sync(KVT_FULL, m1, j);
                    const int pos0 = __shfl_sync(KVT_FULL, m2, j);
                    const int t1 = __shfl_sync(KVT_FULL, m0, (j + 1) & 31), c1 = __shfl_sync(KVT_FULL, m1, (j + 1) & 31);
                    const int p1 = __shfl_sync(KVT_FULL, m2, (j + 1) & 31);
                    if (j + 1 < nb && t1 == t0 + cnt && p1 == pos0 + cnt && cnt + c1 <= QM_ROWS) {
                        cnt += c1;
                        ++j;
                    }
                    const int s = ps;
                    const bool newq = cur != prev;
                    if (lane == 0) {
                        if (pr > 0) mbar_wait(&empty[s], (uint32_t)((pr - 1) & 1));
                        const uint32_t bytes = (uint32_t)(cnt * row_b) + (newq ? (uint32_t)(QG * qb) : 0u);
                        meta[s] = make_int4(cur, t0, cnt, pos0);
                        mbar_arrive_expect_tx(&full[s], bytes);
                        unsigned char* st = smem + (size_t)s * stage_b;
                        const int64_t kv_row = QG > 1 ? (int64_t)cur : (int64_t)(cur / kvg);
                        bulk_g2s(st, keys + kv_row * lane_stride_b + (int64_t)t0 * row_b,
                                 (uint32_t)(cnt * row_b), &full[s]);
                        if (newq) bulk_g2s(st + tile_b, qprep + (int64_t)cur * QG * qb, (uint32_t)(QG * qb), &full[s]);
                    }
                    prev = cur;
                    if (++ps == QM_STAGES) { ps = 0; ++pr; }
                }
                it += nb;
                g += nb;
            }
        }
        if (lane == 0) {
            if (pr > 0) mbar_wait(&empty[ps], (uint32_t)((pr - 1) & 1));
            meta[ps] = make_int4(-1, 0, -1, 0);
            mbar_arrive_expect_tx(&full[ps], 0u);
        }
        return;
    }

    // ---- consumers ----
    const int gid = lane >> 2, tig = lane & 3;
    if constexpr (QG == 1) {
    uint32_t B[R][2][4][2];
    float qt[R], W[R], sp[4];
    int cur = -1;
    // the lane's error bound, accumulated per thread without per-token reductions: the max
    // over its rows of (15|s_g| + |m_g|) for its group and of |est|; combined at the flush
    // into E = 1.001 (u max|est| + sum_g max_rows(15|s_g| + |m_g|) W_g) >= every e(t)
    float gmx[R], amx = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) gmx[r] = 0.f;
    auto lane_bound = [&]() -> float {
        float v = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float gm = gmx[r];
#pragma unroll
            for (int o = 4; o <= 16; o <<= 1) gm = fmaxf(gm, __shfl_xor_sync(KVT_FULL, gm, o));  // rows (gid)
            v = fmaf(gm, W[r], v);
        }
        v += __shfl_xor_sync(KVT_FULL, v, 1);  // groups (tig)
        v += __shfl_xor_sync(KVT_FULL, v, 2);
        float a = amx;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) a = fmaxf(a, __shfl_xor_sync(KVT_FULL, a, o));
        return 1.001f * __fmaf_rn(0x1p-24f, a, v);
    };
    int cs = 0, cr = 0;
    for (;;) {
        const int s = cs;
        mbar_wait(&full[s], (uint32_t)(cr & 1));
        if (++cs == QM_STAGES) { cs = 0; ++cr; }
        const int4 mt = meta[s];
        if (mt.z < 0) break;
        const unsigned char* st = smem + (size_t)s * stage_b;
        if (mt.x != cur) {
            // flush the finished lane's error bound, then load the new lane's digits
            const float e = lane_bound();
            if (lane == 0 && cur >= 0 && e > 0.f)
                atomicMax(reinterpret_cast<unsigned long long*>(err + (int64_t)cur * 4 + 3),
                          (unsigned long long)__double_as_longlong((double)e));
            amx = 0.f;
#pragma unroll
            for (int r = 0; r < R; ++r) gmx[r] = 0.f;
            cur = mt.x;
            const unsigned char* qs = st + tile_b;
            const bool role = (gid >> 1) == tig;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int gq = 4 * r + tig;
#pragma unroll
                for (int S = 0; S < 2; ++S) {
                    const int p = 2 * S + (gid & 1);
                    if (role) {
                        const uint4 x0 = *reinterpret_cast<const uint4*>(qs + gq * 128 + p * 32);
                        const uint4 x1 = *reinterpret_cast<const uint4*>(qs + gq * 128 + p * 32 + 16);
                        B[r][S][0][0] = x0.x; B[r][S][0][1] = x0.y; B[r][S][1][0] = x0.z; B[r][S][1][1] = x0.w;
                        B[r][S][2][0] = x1.x; B[r][S][2][1] = x1.y; B[r][S][3][0] = x1.z; B[r][S][3][1] = x1.w;
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) B[r][S][i][0] = B[r][S][i][1] = 0u;
                    }
                }
                const float2 c2 = *reinterpret_cast<const float2*>(qs + G * 128 + 16 * gq);
                qt[r] = c2.x;
                W[r] = c2.y;
            }
            const float4 s4 = *reinterpret_cast<const float4*>(qs + G * 144);
            sp[0] = s4.x; sp[1] = s4.y; sp[2] = s4.z; sp[3] = s4.w;
        }
        const int cnt = mt.z, pos0 = mt.w, t0 = mt.y;
        float* const o32 = out32 + (int64_t)cur * out_stride + pos0;
        int32_t* const otok = out_tok ? out_tok + (int64_t)cur * out_stride + pos0 : nullptr;
#pragma unroll
        for (int tt = 0; tt < QM_ROWS / 64; ++tt) {
          if (64 * tt + 16 * warp < cnt) {
            const int row0 = 64 * tt + 16 * warp + gid, row1 = row0 + 8;
            float est0, est1;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int gq = 4 * r + tig;
                const uint4 A0 = *reinterpret_cast<const uint4*>(st + row0 * row_b + 16 * gq);
                const uint4 A1 = *reinterpret_cast<const uint4*>(st + row1 * row_b + 16 * gq);
                const uint32_t w0v[4] = {A0.x, A0.y, A0.z, A0.w}, w1v[4] = {A1.x, A1.y, A1.z, A1.w};
                int c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t a0 = w0v[i] & 0x0f0f0f0fu, a2 = (w0v[i] >> 4) & 0x0f0f0f0fu;
                    const uint32_t a1 = w1v[i] & 0x0f0f0f0fu, a3 = (w1v[i] >> 4) & 0x0f0f0f0fu;
                    mma_s8(c0, a0, a1, a2, a3, B[r][0][i][0], B[r][0][i][1]);
                    mma_s8(c1, a0, a1, a2, a3, B[r][1][i][0], B[r][1][i][1]);
                }
                // c0: parts 0,1 / c1: parts 2,3 of group gq; [0],[1] row0, [2],[3] row1.
                // inner = sum_p s_p D_p = s_1 (128 D_0 + D_1) + s_3 (128 D_2 + D_3): the integer
                // pairs are exact in f32 (|.| < 2^24), so 2 conversions and 1 rounding (the fma)
                const float in0 = fmaf(sp[1], (float)(c0[0] * 128 + c0[1]), sp[3] * (float)(c1[0] * 128 + c1[1]));
                const float in1 = fmaf(sp[1], (float)(c0[2] * 128 + c0[3]), sp[3] * (float)(c1[2] * 128 + c1[3]));
                const uint32_t h0 = *reinterpret_cast<const uint32_t*>(st + row0 * row_b + d / 2 + 4 * gq);
                const uint32_t h1 = *reinterpret_cast<const uint32_t*>(st + row1 * row_b + d / 2 + 4 * gq);
                const __half2 p0 = *reinterpret_cast<const __half2*>(&h0), p1 = *reinterpret_cast<const __half2*>(&h1);
                const float sc0 = __low2float(p0), mn0 = __high2float(p0);
                const float sc1 = __low2float(p1), mn1 = __high2float(p1);
                const float e0 = fmaf(sc0, in0, mn0 * qt[r]), e1 = fmaf(sc1, in1, mn1 * qt[r]);
                est0 = r == 0 ? e0 : est0 + e0;
                est1 = r == 0 ? e1 : est1 + e1;
                if (row0 < cnt) gmx[r] = fmaxf(gmx[r], fmaf(15.f, fabsf(sc0), fabsf(mn0)));
                if (row1 < cnt) gmx[r] = fmaxf(gmx[r], fmaf(15.f, fabsf(sc1), fabsf(mn1)));
            }
            // sum over the 4 groups (tig) as a transposed reduction: odd tig keeps row1 and
            // sends row0, even tig the reverse, then one more exchange; the tree is
            // (g0 + g1) + (g2 + g3) for both rows, as before (same bits)
            const bool odd = tig & 1;
            float est = (odd ? est1 : est0) + __shfl_xor_sync(KVT_FULL, odd ? est0 : est1, 1);
            est += __shfl_xor_sync(KVT_FULL, est, 2);
            const int row = odd ? row1 : row0;
            if (tig < 2 && row < cnt) {
                o32[row] = est;
                if (otok) otok[row] = t0 + row;
                amx = fmaxf(amx, fabsf(est));
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    const float e = lane_bound();
    if (lane == 0 && cur >= 0 && e > 0.f)
        atomicMax(reinterpret_cast<unsigned long long*>(err + (int64_t)cur * 4 + 3),
                  (unsigned long long)__double_as_longlong((double)e));
    } else {
    // ---- GQA: heads on the MMA N dimension (module header) ----
    constexpr int NQ = (QG + 3) / 4;  // passes of 4 heads
    uint32_t B[G][2][2];
    float qt[G], W[G], sp[4];
    int cur = -1;
    float emax = 0.f;  // this thread's head of the current pass... per pass below
    float emaxq[NQ];
#pragma unroll
    for (int x = 0; x < NQ; ++x) emaxq[x] = 0.f;
    int cs = 0, cr = 0;
    // head (4 hq + gid / 2) digits for the B operand; head (4 hq + tig) epilogue constants
    auto load_quad = [&](const unsigned char* qs, int hq) {
        const int hb = 4 * hq + (gid >> 1);
        const unsigned char* qb_ = qs + (size_t)(hb < QG ? hb : 0) * qb;
#pragma unroll
        for (int G_ = 0; G_ < G; ++G_) {
#pragma unroll
            for (int S = 0; S < 2; ++S) {
                const int p = 2 * S + (gid & 1);
                const uint2 x = *reinterpret_cast<const uint2*>(qb_ + G_ * 128 + p * 32 + tig * 8);
                B[G_][S][0] = hb < QG ? x.x : 0u;
                B[G_][S][1] = hb < QG ? x.y : 0u;
            }
        }
        const int he = 4 * hq + tig;
        const unsigned char* qe = qs + (size_t)(he < QG ? he : 0) * qb;
#pragma unroll
        for (int G_ = 0; G_ < G; ++G_) {
            const float2 c2 = *reinterpret_cast<const float2*>(qe + G * 128 + 16 * G_);
            qt[G_] = c2.x;
            W[G_] = c2.y;
        }
        const float4 s4 = *reinterpret_cast<const float4*>(qe + G * 144);
        sp[0] = s4.x; sp[1] = s4.y; sp[2] = s4.z; sp[3] = s4.w;
    };
    auto flush = [&]() {
#pragma unroll
        for (int x = 0; x < NQ; ++x) {
            float e2 = emaxq[x];
            // lanes of one tig share a head: reduce over gid (lane bits 2..4)
#pragma unroll
            for (int o = 16; o >= 4; o >>= 1) e2 = fmaxf(e2, __shfl_xor_sync(KVT_FULL, e2, o));
            const int he = 4 * x + tig;
            if (gid == 0 && cur >= 0 && he < QG && e2 > 0.f)
                atomicMax(reinterpret_cast<unsigned long long*>(err + ((int64_t)cur * QG + he) * 4 + 3),
                          (unsigned long long)__double_as_longlong((double)e2));
            emaxq[x] = 0.f;
        }
    };
    (void)emax;
    const unsigned char* qglob = nullptr;
    for (;;) {
        const int s = cs;
        mbar_wait(&full[s], (uint32_t)(cr & 1));
        if (++cs == QM_STAGES) { cs = 0; ++cr; }
        const int4 mt = meta[s];
        if (mt.z < 0) break;
        const unsigned char* st = smem + (size_t)s * stage_b;
        if (mt.x != cur) {
            flush();
            cur = mt.x;
            qglob = qprep + (int64_t)cur * QG * qb;
            load_quad(st + tile_b, 0);
        }
        const int cnt = mt.z, pos0 = mt.w, t0 = mt.y;
#pragma unroll
        for (int tt = 0; tt < QM_ROWS / 64; ++tt) {
          if (64 * tt + 16 * warp < cnt) {
            const int row0 = 64 * tt + 16 * warp + gid, row1 = row0 + 8;
#pragma unroll 1
            for (int hq = 0; hq < NQ; ++hq) {
                if (NQ > 1) load_quad(qglob, hq);  // heads 4 hq.. (L1-resident digit blocks)
                float est0 = 0.f, est1 = 0.f, er0 = 0.f, er1 = 0.f;
#pragma unroll
                for (int G_ = 0; G_ < G; ++G_) {
                    const uint32_t w0 = *reinterpret_cast<const uint32_t*>(st + row0 * row_b + 16 * G_ + 4 * tig);
                    const uint32_t w1 = *reinterpret_cast<const uint32_t*>(st + row1 * row_b + 16 * G_ + 4 * tig);
                    const uint32_t a0 = w0 & 0x0f0f0f0fu, a2 = (w0 >> 4) & 0x0f0f0f0fu;
                    const uint32_t a1 = w1 & 0x0f0f0f0fu, a3 = (w1 >> 4) & 0x0f0f0f0fu;
                    int c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
                    mma_s8(c0, a0, a1, a2, a3, B[G_][0][0], B[G_][0][1]);
                    mma_s8(c1, a0, a1, a2, a3, B[G_][1][0], B[G_][1][1]);
                    // thread tig: head 4 hq + tig, parts 0,1 (c0) and 2,3 (c1), rows gid / gid + 8
                    const float in0 = fmaf(sp[1], (float)(c0[0] * 128 + c0[1]), sp[3] * (float)(c1[0] * 128 + c1[1]));
                    const float in1 = fmaf(sp[1], (float)(c0[2] * 128 + c0[3]), sp[3] * (float)(c1[2] * 128 + c1[3]));
                    const uint32_t h0 = *reinterpret_cast<const uint32_t*>(st + row0 * row_b + d / 2 + 4 * G_);
                    const uint32_t h1 = *reinterpret_cast<const uint32_t*>(st + row1 * row_b + d / 2 + 4 * G_);
                    const __half2 p0 = *reinterpret_cast<const __half2*>(&h0), p1 = *reinterpret_cast<const __half2*>(&h1);
                    const float sc0 = __low2float(p0), mn0 = __high2float(p0);
                    const float sc1 = __low2float(p1), mn1 = __high2float(p1);
                    est0 += fmaf(sc0, in0, mn0 * qt[G_]);
                    est1 += fmaf(sc1, in1, mn1 * qt[G_]);
                    er0 = fmaf(fmaf(15.f, fabsf(sc0), fabsf(mn0)), W[G_], er0);
                    er1 = fmaf(fmaf(15.f, fabsf(sc1), fabsf(mn1)), W[G_], er1);
                }
                const int he = 4 * hq + tig;
                if (he < QG) {
                    const int64_t orow = (int64_t)cur * QG + he;
                    const float e0 = 1.001f * __fmaf_rn(0x1p-24f, fabsf(est0), er0);
                    const float e1 = 1.001f * __fmaf_rn(0x1p-24f, fabsf(est1), er1);
                    float em = 0.f;
                    if (row0 < cnt) { out32[orow * out_stride + pos0 + row0] = est0; em = e0; }
                    if (row1 < cnt) { out32[orow * out_stride + pos0 + row1] = est1; em = fmaxf(em, e1); }
#pragma unroll
                    for (int x = 0; x < NQ; ++x)
                        if (x == hq) emaxq[x] = fmaxf(emaxq[x], em);
                    if (out_tok && he == 0) {
                        const int64_t trow = (int64_t)cur * QG * out_stride + pos0;
                        if (row0 < cnt) out_tok[trow + row0] = t0 + row0;
                        if (row1 < cnt) out_tok[trow + row1] = t0 + row1;
                    }
                }
            }
            if (NQ > 1) load_quad(qglob, 0);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    flush();
    }
}

}  // namespace kvt

using namespace kvt;

extern "C" size_t kvt_i4_qprep_bytes(int64_t n_lanes, int d) {
    if (d != 128 && d != 256) return 0;
    return (size_t)n_lanes * (size_t)qprep_bytes(d);
}

extern "C" int kvt_i4_qprep(const void* q, int q_dtype, int64_t n_lanes, int d, void* out, void* stream) {
    if (d != 128 && d != 256) return KVT_ERR_SHAPE;
    if (n_lanes <= 0) return n_lanes == 0 ? KVT_OK : KVT_ERR_ARG;
    if (!q || !out || ((uintptr_t)out % 16)) return KVT_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int wpb = 8;
    const unsigned grid = (unsigned)((n_lanes + wpb - 1) / wpb);
    if (q_dtype == KVT_F32)
        launch_pdl(qprep_kernel<float>, dim3(grid), dim3(32 * wpb), 0, st, (const float*)q, n_lanes, d, (unsigned char*)out);
    else if (q_dtype == KVT_F64)
        launch_pdl(qprep_kernel<double>, dim3(grid), dim3(32 * wpb), 0, st, (const double*)q, n_lanes, d,
                   (unsigned char*)out);
    else return KVT_ERR_DTYPE;
    return kvt_check_launch();
}

template <int R, int QG>
static int launch_i4mma(const void* keys, int64_t n_rows, int64_t ls_b, const int32_t* items, int64_t item_stride,
                        const int32_t* n_items, const void* qprep, float* os, int32_t* ot, int64_t ostr, double* err,
                        cudaStream_t st) {
    constexpr int d = 128 * R, G = 4 * R, row_b = d / 2 + G * 4, tile_b = QM_ROWS * row_b, qb = G * 144 + 16;
    constexpr int stage_b = (tile_b + QG * qb + 15) / 16 * 16;
    const size_t smem = (size_t)QM_STAGES * stage_b;
    KVT_PER_DEVICE(bool, configured);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(score_i4mma_kernel<R, QG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        configured = true;
    }
    const int sms = kvt::sm_count();
    KVT_PER_DEVICE(int, per_sm);
    if (!per_sm) per_sm = resident_per_sm(score_i4mma_kernel<R, QG>, QM_THREADS, smem, 4);
    launch_pdl(score_i4mma_kernel<R, QG>, dim3(sms * per_sm), dim3(QM_THREADS), smem, st, (const unsigned char*)keys, ls_b,
               (int)n_rows, items, item_stride, n_items, (const unsigned char*)qprep, os, ot, ostr, err,
               kv_group_current());
    return kvt_check_launch();
}

extern "C" int kvt_cand_score_i4mma(const void* q, int q_dtype, const void* keys, int64_t n_lanes, int64_t lane_stride,
                                    int d, const int32_t* items, int64_t item_stride, const int32_t* n_items,
                                    float* cand_score32, int32_t* cand_tok, int64_t cand_stride, double* err,
                                    void* qprep_ws, void* stream) {
    if (d != 128 && d != 256) return KVT_ERR_SHAPE;
    if (n_lanes <= 0) return n_lanes == 0 ? KVT_OK : KVT_ERR_ARG;
    if (!keys || !items || !n_items || !cand_score32 || !err || !qprep_ws) return KVT_ERR_ARG;
    if (((uintptr_t)keys % 16) || (lane_stride % 16) || n_lanes > INT32_MAX) return KVT_ERR_SHAPE;
    // GQA union mode (cand_group g > 1): items per KV lane; g must divide n_lanes (query lanes)
    const int qg = cand_group_current();
    if (qg > 1 && (qg > 8 || n_lanes % qg || qg != kv_group_current())) return KVT_ERR_ARG;
    if (q) {  // q == nullptr: qprep_ws already holds the digits (kvt_select_attend runs kvt_i4_qprep on a side stream)
        int rc = kvt_i4_qprep(q, q_dtype, n_lanes, d, qprep_ws, stream);
        if (rc) return rc;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = n_lanes / qg;
#define KVT_QM(RR, QQ) launch_i4mma<RR, QQ>(keys, rows, lane_stride, items, item_stride, n_items, qprep_ws, \
                                            cand_score32, cand_tok, cand_stride, err, st)
    if (qg == 1) return d == 128 ? KVT_QM(1, 1) : KVT_QM(2, 1);
    if (qg == 2) return d == 128 ? KVT_QM(1, 2) : KVT_QM(2, 2);
    if (qg <= 4) return qg == 4 ? (d == 128 ? KVT_QM(1, 4) : KVT_QM(2, 4)) : KVT_ERR_ARG;
    return qg == 8 ? (d == 128 ? KVT_QM(1, 8) : KVT_QM(2, 8)) : KVT_ERR_ARG;
#undef KVT_QM
}
