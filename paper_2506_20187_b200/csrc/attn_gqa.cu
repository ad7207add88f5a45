// attn_gqa.cu -- K7 for GQA groups over INT4 values: one pass over the UNION of the group's
// selections, the P.V product on the tensor cores with the group's heads as the MMA rows.
//
// engine.py:145-154 attention_output = softmax(q.K_sel^T / sqrt d) . V_sel, per query head.
// The reference replicates each KV head per query head (adapters.py:121-136), so g query
// heads sharing a KV head read, dequantise and multiply the same value rows g times.  Here a
// KV lane's value rows are streamed once for its g heads, in two launches:
//   plan  (one CTA per KV lane x 2048-token window): every head's selected tokens in the
//         window (a warp-wide 32-ary lower_bound in its ascending selection) as bitmaps, their
//         OR = the union rows (ascending token offsets, popcount prefix), and per union row the
//         g softmax weights w_h = exp((s_h - m_wh) / sqrt d) relative to the window max m_wh (0
//         where head h did not select the row), written to scratch with the window's count;
//   pv    (one CTA per KV lane x range of windows, 4 warps): the union rows' 80 B INT4 value
//         records stream through a per-warp cp.async ring, 16 rows per tile, and
//             o_h[j] = sum_t w_h(t) (s_t,G(j) (c_t,j - 8) + (m_t,G(j) + 8 s_t,G(j)))
//         runs on mma.sync m16n8k16 (f16 in, f32 accumulate): A = the weights times the group's
//         scale (x 2^12), rows 2h / 2h + 1 = their f16 high / low parts, so the product keeps
//         ~22 bits; B = the centred codes c - 8 as exact f16 integers (nibbles -> 1024 + c by one
//         LOP3, minus 1032 by one HSUB2); 16 MMAs per 16 rows cover d = 128 for every head at once.  The
//         min term sum_t w_h(t) m_t,G is a per-(head, group) scalar on the CUDA cores.  Each
//         warp keeps flash-decoding state per head (running max over its tiles' windows); the
//         warps and then the ranges (ticket: the last range CTA of the KV lane) are merged.
// Values are read once per KV lane instead of once per query head, and dequantised once; the
// staging no longer sits between the loads and the MMAs (the pv loop is one continuous ring).
#include "common.cuh"

namespace kvt {

constexpr int GQ_WARPS = 4;
constexpr int GQ_THREADS = GQ_WARPS * 32;
constexpr int GQ_S = 6;              // ring slots per warp (16 rows x 80 B each)
constexpr int GQ_ROWB = 80;          // INT4 record bytes at d = 128
constexpr int GQ_SLOT = 16 * GQ_ROWB;
constexpr int GQ_SSLOT = GQ_SLOT + 16 * 4 * 4 + 4 * 8 + 16;  // + weights [16][4] f32, head maxima, header
constexpr float GQ_ASCALE = 4096.f;  // A pre-scale: keeps the f16 low parts normal
constexpr int GQ_WIN = 2048;         // tokens staged per window (bitmaps, slots, weights)

__device__ __forceinline__ void gq_cp16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void gq_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void gq_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void mma_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
    return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
}

// first index i in [0, n) with tok[i] >= target (tok ascending); whole warp, ~3 probes
__device__ __forceinline__ int warp_lower_bound(const int32_t* __restrict__ tok, int n, int target, int lane) {
    int lo = 0, hi = n;
    while (hi - lo > 32) {
        const int stride = (hi - lo + 31) / 32;
        const int pos = lo + lane * stride;
        const bool below = pos < hi && tok[pos] < target;
        const int c = __popc(__ballot_sync(KVT_FULL, below));  // probes below target form a prefix
        const int nlo = c == 0 ? lo : lo + (c - 1) * stride;
        hi = c == 32 ? hi : kvt::imin(hi, lo + c * stride);
        lo = nlo;
    }
    const int pos = lo + lane;
    const bool below = pos < hi && tok[pos] < target;
    return lo + __popc(__ballot_sync(KVT_FULL, below));
}

// merge of one query lane's range partials (as attn_finish in runs_attn.cu, with the lane
// count explicit and empty partials skipped); run by the last-arriving CTA of the KV lane
__device__ void gq_merge(double* __restrict__ part, int splits, int d, int64_t li, int64_t n_lanes,
                         float* __restrict__ out, double* __restrict__ out64, double scale) {
    __shared__ double s_scale[64];
    __shared__ double s_den, s_M;
    const double* P = part + li * splits * (int64_t)(d + 2);
    if (threadIdx.x < 32) {
        double M = -INFINITY;
        for (int s = threadIdx.x; s < splits; s += 32)
            if (__ldcg(P + s * (d + 2) + 1) > 0) M = fmax(M, __ldcg(P + s * (d + 2)));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) M = fmax(M, __shfl_xor_sync(KVT_FULL, M, off));
        double den = 0.0;
        for (int s = threadIdx.x; s < splits; s += 32) {
            const double ls = __ldcg(P + s * (d + 2) + 1);
            const double sc = ls > 0 ? exp((__ldcg(P + s * (d + 2)) - M) * scale) : 0.0;
            s_scale[s] = sc;
            den += sc * ls;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) den += __shfl_xor_sync(KVT_FULL, den, off);
        if (threadIdx.x == 0) { s_den = den; s_M = M; }
    }
    __syncthreads();
    const double den = s_den;
    if (threadIdx.x == 0) {  // per-lane (m, l) of the merged softmax, for cross-shard merges
        double* lse = part - 2 * n_lanes;
        lse[2 * li] = s_M;
        lse[2 * li + 1] = den;
    }
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < splits; ++s)
            if (s_scale[s] != 0.0) acc += s_scale[s] * __ldcg(P + s * (d + 2) + 2 + j);
        const double r = den > 0 ? acc / den : 0.0;
        if (out) out[li * d + j] = (float)r;
        if (out64) out64[li * d + j] = r;
    }
    __syncthreads();
}


// ---- scratch layout of the plan (kvt_attn_gqa_scratch_bytes) ---------------------------------
struct GqPlan {
    int32_t* cnt;    // [n_kv][n_win] union rows of the window
    double* mx;      // [n_kv][n_win][G] window max score per head (-inf: none)
    uint16_t* off;   // [n_kv][n_win][W] union rows' token offsets in the window, ascending
    float* wt;       // [n_kv][n_win][W][G] weights relative to the window max (0: not selected)
};
__host__ __device__ inline size_t gq_al(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ inline GqPlan gq_carve(void* base, int64_t n_kv, int64_t n_win, int G) {
    char* p = (char*)base;
    GqPlan P;
    const size_t nw = (size_t)n_kv * n_win;
    P.cnt = (int32_t*)p;
    p += gq_al(nw * 4);
    P.mx = (double*)p;
    p += gq_al(nw * G * 8);
    P.off = (uint16_t*)p;
    p += gq_al(nw * GQ_WIN * 2);
    P.wt = (float*)p;
    return P;
}
inline size_t gq_scratch_bytes(int64_t n_kv, int64_t n_win, int G) {
    const size_t nw = (size_t)n_kv * n_win;
    return gq_al(nw * 4) + gq_al(nw * G * 8) + gq_al(nw * GQ_WIN * 2) + gq_al(nw * GQ_WIN * G * 4);
}

#ifndef KVT_GQ_WPC
#define KVT_GQ_WPC 1
#endif
#ifndef KVT_GQ_PLAN_MINB
#define KVT_GQ_PLAN_MINB 1
#endif
constexpr int GQ_WPC = KVT_GQ_WPC;  // windows per plan CTA (one lower_bound, then a forward scan)

template <int G>
__global__ void __launch_bounds__(GQ_THREADS, KVT_GQ_PLAN_MINB) gqa_plan_kernel(const int32_t* __restrict__ sel_tok,
                                                              const double* __restrict__ sel_score,
                                                              const int32_t* __restrict__ n_sel, int64_t sel_stride,
                                                              int64_t n_win, double scale, GqPlan P) {
    pdl_entry();
    constexpr int W = GQ_WIN, NW = W / 32;
    constexpr int SCAN = 4;
    __shared__ uint32_t bm[G * NW];  // per-head bitmaps of the window
    __shared__ uint32_t ubm[NW];
    __shared__ int upre[NW];
    __shared__ int s_a[G], s_b[G];
    __shared__ double s_m[G];
    __shared__ int scan_sh[33];
    __shared__ int s_ucnt;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t kv = blockIdx.y;
    const int64_t win0 = (int64_t)blockIdx.x * GQ_WPC, win1 = kvt::imin(n_win, win0 + GQ_WPC);
    const double sl2 = scale * 1.4426950408889634;
    // each head's first entry at or after the CTA's first window (one search per CTA)
    for (int h = warp; h < G; h += GQ_WARPS) {
        const int64_t li = kv * G + h;
        const int a = warp_lower_bound(sel_tok + li * sel_stride, n_sel[li], (int)(win0 * W), lane);
        if (lane == 0) s_b[h] = a;
    }
    for (int64_t win = win0; win < win1; ++win) {
        const int T0 = (int)(win * W);
        for (int i = tid; i < G * NW; i += GQ_THREADS) bm[i] = 0u;
        __syncthreads();
        // 1. each head's window entries (a prefix of its remaining ones) -> bitmap and max
        for (int h = warp; h < G; h += GQ_WARPS) {
            const int64_t li = kv * G + h;
            const int n = n_sel[li];
            const int32_t* tk = sel_tok + li * sel_stride;
            const double* sc = sel_score + li * sel_stride;
            const int a = s_b[h];
            int j = a;
            double mx = -INFINITY;
            for (;;) {
                int t[SCAN];
                double v[SCAN];
#pragma unroll
                for (int u = 0; u < SCAN; ++u) {  // ids and scores issued together: one latency
                    const int pos = j + 32 * u + lane;
                    t[u] = pos < n ? tk[pos] - T0 : INT_MAX;
                    v[u] = pos < n ? sc[pos] : -INFINITY;
                }
                int taken = 0;
#pragma unroll
                for (int u = 0; u < SCAN; ++u) {
                    const bool in = t[u] < W;
                    taken += __popc(__ballot_sync(KVT_FULL, in));
                    if (in) {
                        atomicOr(&bm[h * NW + (t[u] >> 5)], 1u << (t[u] & 31));
                        mx = fmax(mx, v[u]);
                    }
                }
                j += taken;
                if (taken < 32 * SCAN) break;
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(KVT_FULL, mx, o));
            if (lane == 0) { s_a[h] = a; s_b[h] = j; s_m[h] = mx; }
        }
        __syncthreads();
        // 2. union rows: OR of the bitmaps, popcount prefix
        for (int w = tid; w < NW; w += GQ_THREADS) {
            uint32_t u = 0;
#pragma unroll
            for (int h = 0; h < G; ++h) u |= bm[h * NW + w];
            ubm[w] = u;
        }
        __syncthreads();
        {
            int tot;
            // prefix over the NW = 64 words: thread tid owns words 2 tid, 2 tid + 1
            const int w0 = 2 * tid, w1 = 2 * tid + 1;
            const int c0 = w0 < NW ? __popc(ubm[w0]) : 0, c1 = w1 < NW ? __popc(ubm[w1]) : 0;
            const int ex = block_excl_scan<int>(c0 + c1, scan_sh, tot);
            if (w0 < NW) upre[w0] = ex;
            if (w1 < NW) upre[w1] = ex + c0;
            if (tid == 0) s_ucnt = tot;
        }
        __syncthreads();
        const int ucnt = s_ucnt;
        const size_t wb = (size_t)(kv * n_win + win);
        uint16_t* off = P.off + wb * W;
        for (int w = tid; w < NW; w += GQ_THREADS) {
            uint32_t x = ubm[w];
            int sl = upre[w];
            while (x) {
                const int bit = __ffs(x) - 1;
                x &= x - 1;
                off[sl++] = (uint16_t)(w * 32 + bit);
            }
        }
        float* dstw = P.wt + wb * W * G;
        if constexpr (G % 4 == 0) {
            float4* dz = reinterpret_cast<float4*>(dstw);
            for (int i = tid; i < ucnt * G / 4; i += GQ_THREADS) dz[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (int i = tid; i < ucnt * G; i += GQ_THREADS) dstw[i] = 0.f;
        }
        __syncthreads();  // zeros before the scatter (global writes of the block are ordered by it)
        // 3. weights of each head's entries at their union rows (entries just read: L1 hits)
        for (int h = warp; h < G; h += GQ_WARPS) {
            const int64_t li = kv * G + h;
            const int32_t* tk = sel_tok + li * sel_stride;
            const double* sc = sel_score + li * sel_stride;
            const double mh = s_m[h];
            for (int j = s_a[h] + lane; j < s_b[h]; j += 32) {
                const int t = tk[j] - T0;
                const int w = t >> 5;
                const int slot = upre[w] + __popc(ubm[w] & ((1u << (t & 31)) - 1u));
                dstw[slot * G + h] = exp2f((float)((sc[j] - mh) * sl2));
            }
        }
        if (tid < G) P.mx[wb * G + tid] = s_m[tid];
        if (tid == 0) P.cnt[wb] = ucnt;
        __syncthreads();  // wtab / bitmaps / s_* reused by the next window
    }
}

template <int G>  // heads per KV lane (2 or 4): rows 2h, 2h + 1 of A
__global__ void __launch_bounds__(GQ_THREADS, 4) gqa_pv_kernel(
    const unsigned char* __restrict__ values, int64_t lane_stride_b, int64_t n_q, int64_t n_win, int wins_per,
    int splits, int64_t n_tok_ctx, GqPlan P, double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out,
    double* __restrict__ out64, double scale) {
    pdl_entry();
    constexpr int d = 128;
    constexpr int MAXW = 256;  // windows per range (host guarantees)
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char* ring = smem;  // [warps][S][16 x 80 B]
    __shared__ int s_tpre[MAXW + 1];
    __shared__ float s_o[GQ_WARPS][G][d];
    __shared__ float s_om[GQ_WARPS][G][4];
    __shared__ double s_wm[GQ_WARPS][G];
    __shared__ float s_wl[GQ_WARPS][G];
    __shared__ int scan_sh[33];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t kv = blockIdx.y;
    const int rg = blockIdx.x;
    const int64_t w0 = (int64_t)rg * wins_per, w1 = kvt::imin(n_win, w0 + wins_per);
    const int nwin = (int)kvt::imax(0, w1 - w0);
    const double sl2 = scale * 1.4426950408889634;
    const int gid = lane >> 2, tig = lane & 3;
    const int hA = gid >> 1;             // head of A row gid (rows 2G.. stay zero)
    const bool lo_part = gid & 1;
    const unsigned char* vbase = values + kv * lane_stride_b;
    unsigned char* wring = ring + (size_t)warp * GQ_S * GQ_SSLOT;
    const uint32_t wring_a = (uint32_t)__cvta_generic_to_shared(wring);
    const size_t wbase = (size_t)(kv * n_win + w0);

    // tiles of the range's windows: exclusive prefix of ceil(cnt / 16)
    {
        const int c0 = tid < nwin ? (P.cnt[wbase + tid] + 15) / 16 : 0;
        const int c1 = tid + GQ_THREADS < nwin ? (P.cnt[wbase + tid + GQ_THREADS] + 15) / 16 : 0;
        int tot;
        const int e0 = block_excl_scan<int>(c0, scan_sh, tot);
        if (tid < nwin) s_tpre[tid] = e0;
        const int t0 = tot;
        const int e1 = block_excl_scan<int>(c1, scan_sh, tot);
        if (tid + GQ_THREADS < nwin) s_tpre[tid + GQ_THREADS] = t0 + e1;
        if (tid == 0) s_tpre[nwin] = t0 + tot;
    }
    __syncthreads();
    const int ntile = s_tpre[nwin];
    const int my_tiles = ntile > warp ? (ntile - warp + GQ_WARPS - 1) / GQ_WARPS : 0;  // tiles warp, warp + 4, ...

    // window of a tile: last wi with s_tpre[wi] <= tile (tiles of one warp only move forward)
    auto window_of = [&](int tile, int from) -> int {
        int wi = from;
        while (s_tpre[wi + 1] <= tile) ++wi;
        return wi;
    };
    // Tile metadata is loaded one iteration before its copies are issued (registers), so no
    // global latency sits between the ring and the MMAs: the copies carry the V records, the
    // tile's weights and a small header (row count, the window max of each head).
    int n_tok[3];          // this lane's 3 pieces: token of its row
    int n_cnt = 0;         // rows of the tile's window
    int n_u0 = 0;          // first union row of the tile
    size_t n_wb = 0;
    double n_mx = -INFINITY;  // lane h < G: window max of head h
    int wi_meta = 0;
    auto load_meta = [&](int tile) {
        wi_meta = window_of(tile, wi_meta);
        const int ti = tile - s_tpre[wi_meta];
        n_wb = wbase + wi_meta;
        n_cnt = P.cnt[n_wb];
        n_u0 = ti * 16;
        const int T0 = (int)((w0 + wi_meta) * GQ_WIN);
        const uint16_t* off = P.off + n_wb * GQ_WIN;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int p = 32 * k + lane;
            const int r = (p < 80 ? p : 0) / 5;
            // rows past the window's count hold stale offsets (< W): a readable record, weight 0
            // (clamped to the context; no dependence on the count load)
            n_tok[k] = (int)kvt::imin((int64_t)(T0 + (int)off[n_u0 + r]), n_tok_ctx - 1);
        }
        n_mx = lane < G ? P.mx[n_wb * G + lane] : -INFINITY;
    };
    constexpr int WB = 16 * G * 4;  // weight bytes per tile
    auto issue = [&](uint32_t dst, unsigned char* sdst) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int p = 32 * k + lane;
            if (p < 80) {
                const int r = p / 5, pc = p % 5;
                gq_cp16(dst + r * GQ_ROWB + pc * 16, vbase + (int64_t)n_tok[k] * GQ_ROWB + pc * 16);
            }
        }
        if (lane < WB / 16)  // rows n_u0 .. n_u0 + 15 of the window's weight table (contiguous)
            gq_cp16(dst + GQ_SLOT + 16 * lane,
                    P.wt + (n_wb * GQ_WIN + n_u0) * G + 4 * lane);
        if (lane < G) reinterpret_cast<double*>(sdst + GQ_SLOT + WB)[lane] = n_mx;
        if (lane == 0) reinterpret_cast<int*>(sdst + GQ_SLOT + WB + 8 * G)[0] = n_cnt - n_u0;  // valid rows
    };

    float D[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) D[j][0] = D[j][1] = D[j][2] = D[j][3] = 0.f;
    float om[4] = {0.f, 0.f, 0.f, 0.f};  // sum_t w_h(t) m_t,G for head hA (hi-part rows)
    double M = -INFINITY;                // running max of head hA over this warp's tiles
    float l = 0.f;                       // running softmax denominator of head hA (hi rows)

    if (my_tiles > 0) load_meta(warp);
#pragma unroll
    for (int j = 0; j < GQ_S - 1; ++j) {
        if (j < my_tiles) {
            issue(wring_a + j * GQ_SSLOT, wring + j * GQ_SSLOT);
            if (j + 1 < my_tiles) load_meta(warp + (j + 1) * GQ_WARPS);
        }
        gq_commit();
    }
    for (int it = 0; it < my_tiles; ++it) {
        const int jn = it + GQ_S - 1;
        if (jn < my_tiles) {
            issue(wring_a + (jn % GQ_S) * GQ_SSLOT, wring + (jn % GQ_S) * GQ_SSLOT);
            if (jn + 1 < my_tiles) load_meta(warp + (jn + 1) * GQ_WARPS);
        }
        gq_commit();
        gq_wait<GQ_S - 1>();
        __syncwarp();
        const unsigned char* slot = wring + (it % GQ_S) * GQ_SSLOT;
        const float* wsl = reinterpret_cast<const float*>(slot + GQ_SLOT);
        const double mw = hA < G ? reinterpret_cast<const double*>(slot + GQ_SLOT + WB)[hA] : -INFINITY;
        const int nvalid = reinterpret_cast<const int*>(slot + GQ_SLOT + WB + 8 * G)[0];
        // this tile's window max for head hA: rescale the running state when it rises
        float f = 0.f;  // weight factor exp(mw - M) for this tile
        if (mw > M) {
            const float rs = M == -INFINITY ? 0.f : exp2f((float)((M - mw) * sl2));
#pragma unroll
            for (int j = 0; j < 16; ++j) { D[j][0] *= rs; D[j][1] *= rs; }
#pragma unroll
            for (int Gq = 0; Gq < 4; ++Gq) om[Gq] *= rs;
            l *= rs;
            M = mw;
            f = 1.f;
        } else if (mw > -INFINITY) {
            f = exp2f((float)((mw - M) * sl2));
        }
        auto wgt = [&](int r) -> float { return (hA < G && r < nvalid) ? wsl[r * G + hA] * f : 0.f; };
        const int r0 = 2 * tig, r1 = 2 * tig + 1, r8 = 2 * tig + 8, r9 = 2 * tig + 9;
        const float wA0 = wgt(r0), wA1 = wgt(r1), wA8 = wgt(r8), wA9 = wgt(r9);
        if (!lo_part) l += wA0 + wA1 + wA8 + wA9;

#pragma unroll
        for (int Gq = 0; Gq < 4; ++Gq) {
            const __half2 p0 = *reinterpret_cast<const __half2*>(slot + r0 * GQ_ROWB + 64 + 4 * Gq);
            const __half2 p1 = *reinterpret_cast<const __half2*>(slot + r1 * GQ_ROWB + 64 + 4 * Gq);
            const __half2 p8 = *reinterpret_cast<const __half2*>(slot + r8 * GQ_ROWB + 64 + 4 * Gq);
            const __half2 p9 = *reinterpret_cast<const __half2*>(slot + r9 * GQ_ROWB + 64 + 4 * Gq);
            const float s0 = __low2float(p0), s1 = __low2float(p1), s8 = __low2float(p8), s9 = __low2float(p9);
            // centred codes: x = (c - 8) s + (m + 8 s), so neither sum carries the other's
            // magnitude (the uncentred split cancels to ~1e-3 of its terms over long selections)
            if (!lo_part)
                om[Gq] += wA0 * fmaf(8.f, s0, __high2float(p0)) + wA1 * fmaf(8.f, s1, __high2float(p1)) +
                          wA8 * fmaf(8.f, s8, __high2float(p8)) + wA9 * fmaf(8.f, s9, __high2float(p9));
            auto split = [&](float v) -> __half {
                const __half hi = __float2half_rn(v);
                return lo_part ? __float2half_rn(v - __half2float(hi)) : hi;
            };
            const uint32_t a0 = pack_h2(split(wA0 * s0 * GQ_ASCALE), split(wA1 * s1 * GQ_ASCALE));
            const uint32_t a2 = pack_h2(split(wA8 * s8 * GQ_ASCALE), split(wA9 * s9 * GQ_ASCALE));
            const int wo = 4 * (4 * Gq + (gid >> 1));
            const uint32_t c0 = *reinterpret_cast<const uint32_t*>(slot + r0 * GQ_ROWB + wo);
            const uint32_t c1 = *reinterpret_cast<const uint32_t*>(slot + r1 * GQ_ROWB + wo);
            const uint32_t c8 = *reinterpret_cast<const uint32_t*>(slot + r8 * GQ_ROWB + wo);
            const uint32_t c9 = *reinterpret_cast<const uint32_t*>(slot + r9 * GQ_ROWB + wo);
            const uint32_t sel = (gid & 1) ? 0x7632u : 0x5410u;
            const uint32_t x01 = __byte_perm(c0, c1, sel), x89 = __byte_perm(c8, c9, sel);
            const __half2 k1032 = __halves2half2(__ushort_as_half(0x6408), __ushort_as_half(0x6408));  // 1024 + 8
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t e01 = ((x01 >> (4 * q)) & 0x000f000fu) | 0x64006400u;
                const uint32_t e89 = ((x89 >> (4 * q)) & 0x000f000fu) | 0x64006400u;
                const __half2 h01 = __hsub2(*reinterpret_cast<const __half2*>(&e01), k1032);
                const __half2 h89 = __hsub2(*reinterpret_cast<const __half2*>(&e89), k1032);
                mma_f16(D[4 * Gq + q], a0, 0u, a2, 0u, *reinterpret_cast<const uint32_t*>(&h01),
                        *reinterpret_cast<const uint32_t*>(&h89));
            }
        }
        __syncwarp();
    }
    gq_wait<0>();

    // ---- per-warp head state -> shared; combine warps (flash-decoding) -> range partials ----
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) D[j][e] += __shfl_xor_sync(KVT_FULL, D[j][e], 4);  // hi + lo rows
#pragma unroll
    for (int Gq = 0; Gq < 4; ++Gq) {
        float v = om[Gq];
        v += __shfl_xor_sync(KVT_FULL, v, 1);
        v += __shfl_xor_sync(KVT_FULL, v, 2);
        om[Gq] = v;
    }
    l += __shfl_xor_sync(KVT_FULL, l, 1);
    l += __shfl_xor_sync(KVT_FULL, l, 2);
    if (!lo_part && hA < G) {
        const float inv = 1.f / GQ_ASCALE;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int dA = 32 * (j >> 2) + 8 * tig + (j & 3);
            s_o[warp][hA][dA] = D[j][0] * inv;
            s_o[warp][hA][dA + 4] = D[j][1] * inv;
        }
        if (tig == 0) {
#pragma unroll
            for (int Gq = 0; Gq < 4; ++Gq) s_om[warp][hA][Gq] = om[Gq];
            s_wm[warp][hA] = M;
            s_wl[warp][hA] = l;
        }
    }
    __syncthreads();
    for (int h = 0; h < G; ++h) {
        double Mh = -INFINITY;
#pragma unroll
        for (int w = 0; w < GQ_WARPS; ++w) Mh = fmax(Mh, s_wm[w][h]);
        float sw[GQ_WARPS];
        float lsum = 0.f;
#pragma unroll
        for (int w = 0; w < GQ_WARPS; ++w) {
            sw[w] = s_wm[w][h] == -INFINITY ? 0.f : exp2f((float)((s_wm[w][h] - Mh) * sl2));
            lsum += sw[w] * s_wl[w][h];
        }
        const int64_t li = kv * G + h;
        double* Pp = part + (li * splits + rg) * (int64_t)(d + 2);
        for (int j = tid; j < d; j += GQ_THREADS) {
            float acc = 0.f;
#pragma unroll
            for (int w = 0; w < GQ_WARPS; ++w) acc += sw[w] * (s_o[w][h][j] + s_om[w][h][j >> 5]);
            Pp[2 + j] = (double)acc;
        }
        if (tid == 0) {
            Pp[0] = Mh;
            Pp[1] = (double)lsum;
        }
    }
    // ---- one ticket per KV lane: the last range CTA merges the group's heads ----
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned t = atomicAdd(&tickets[kv * G], 1u);
        s_last = (t == (unsigned)splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int h = 0; h < G; ++h) gq_merge(part, splits, d, kv * G + h, n_q, out, out64, scale);
    if (tid == 0) tickets[kv * G] = 0;
}

}  // namespace kvt

using namespace kvt;

extern "C" size_t kvt_attn_gqa_scratch_bytes(int64_t n_lanes, int kvg, int64_t n_ctx) {
    if (kvg < 2 || n_lanes % kvg || n_ctx <= 0) return 0;
    return gq_scratch_bytes(n_lanes / kvg, (n_ctx + GQ_WIN - 1) / GQ_WIN, kvg);
}

// GQA INT4 attention over the group's union (kv_group g in {2, 4}, d = 128, tokens < n_ctx):
// plan + pv launches.  scratch: kvt_attn_gqa_scratch_bytes.  Returns KVT_ERR_ARG when the
// shape is not covered (the caller then runs the per-lane kernel).
extern "C" int kvt_sparse_decode_attn_gqa(const void* values, int64_t n_lanes, int64_t lane_stride_b, int d, int kvg,
                                          int64_t n_ctx, const int32_t* sel_tok, const double* sel_score,
                                          const int32_t* n_sel, int64_t sel_stride, double logit_scale, void* ws,
                                          void* scratch, size_t scratch_bytes, float* out, double* out64,
                                          void* stream) {
    if (!values || !sel_tok || !sel_score || !n_sel || !ws || !scratch || (!out && !out64)) return KVT_ERR_ARG;
    if (d != 128 || (kvg != 2 && kvg != 4) || n_lanes <= 0 || n_lanes % kvg || n_ctx <= 0) return KVT_ERR_ARG;
    if (((uintptr_t)values % 16) || (lane_stride_b % 16)) return KVT_ERR_SHAPE;
    if (scratch_bytes < kvt_attn_gqa_scratch_bytes(n_lanes, kvg, n_ctx)) return KVT_ERR_OOM;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n_kv = n_lanes / kvg;
    const int64_t n_win = (n_ctx + GQ_WIN - 1) / GQ_WIN;
    if (n_kv > 65535 || n_win > 65535 * 64) return KVT_ERR_ARG;
    GqPlan P = gq_carve(scratch, n_kv, n_win, kvg);
    // ranges: at most 4 CTAs per SM over the KV lanes (one wave), <= 64 ranges, <= 256 windows each
    int64_t want = (4LL * kvt::sm_count()) / n_kv;
    want = kvt::imax(1, kvt::imin(kvt::imin(want, 64), n_win));
    int wins_per = (int)((n_win + want - 1) / want);
    if (wins_per > 256) return KVT_ERR_ARG;
    const int splits = (int)((n_win + wins_per - 1) / wins_per);
    unsigned int* tickets = (unsigned int*)ws;
    double* part = (double*)((char*)ws + (((size_t)n_lanes * 4 + 255) & ~(size_t)255)) + 2 * n_lanes;
    const size_t smem_pv = (size_t)GQ_WARPS * GQ_S * GQ_SSLOT;
#define KVT_GQ(GG)                                                                                                   \
    do {                                                                                                             \
        launch_pdl(gqa_plan_kernel<GG>, dim3((unsigned)((n_win + GQ_WPC - 1) / GQ_WPC), (unsigned)n_kv),             \
                   dim3(GQ_THREADS), 0, st,                                                                  \
                   sel_tok, sel_score, n_sel, sel_stride, n_win, logit_scale, P);                                    \
        launch_pdl(gqa_pv_kernel<GG>, dim3((unsigned)splits, (unsigned)n_kv), dim3(GQ_THREADS), smem_pv, st,         \
                   (const unsigned char*)values, lane_stride_b, n_lanes, n_win, wins_per, splits, n_ctx, P, part,    \
                   tickets,                                                                                          \
                   out, out64, logit_scale);                                                                         \
    } while (0)
    if (kvg == 2) KVT_GQ(2);
    else KVT_GQ(4);
#undef KVT_GQ
    return kvt_check_launch();
}
