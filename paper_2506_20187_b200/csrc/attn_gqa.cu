// attn_gqa.cu -- K7 for GQA groups over INT4 values: one pass over the UNION of the group's
// selections, the P.V product on the tensor cores with the group's heads as the MMA rows.
//
// engine.py:145-154 attention_output = softmax(q.K_sel^T / sqrt d) . V_sel, per query head.
// The reference replicates each KV head per query head (adapters.py:121-136), so g query
// heads sharing a KV head read (and here would dequantise) the same value rows g times.
// This kernel walks the KV lane's tokens in ranges of R and, per range:
//   1. stages every head's selected tokens in the range (a warp-wide 32-ary lower_bound in
//      each head's ascending selection) as per-head bitmaps, with the head's max score;
//   2. ORs them into the union, assigns union slots (popcount prefix) and scatters each
//      head's softmax weight w_h(t) = exp((s_h(t) - m_h) / sqrt d) into a [slot][head]
//      table (0 where the head did not select t);
//   3. streams the union's value records (80 B INT4 rows: 64 B of codes, four fp16 (scale,
//      min) pairs) through a per-warp cp.async ring, 16 rows per step, and accumulates
//          o_h[j] = sum_t w_h(t) (s_t,G(j) c_t,j + m_t,G(j))
//      with mma.sync m16n8k16 (f16 in, f32 accumulate): A = the weights times the group's
//      scale (x 2^12), rows 2h / 2h + 1 = their f16 high / low parts, so the product keeps
//      ~22 bits (g <= 4 heads fill rows 0..7); B = the codes as exact f16 integers (nibbles -> 1024 + c by
//      one LOP3, minus 1024 by one HSUB2), the MMA's K = 16 union rows, N = 8 dims of one
//      quantisation group, 16 MMAs per 16 rows cover d = 128 for every head at once.  The
//      min term sum_t w_h(t) m_t,G is a per-(head, group) scalar on the CUDA cores.
//   4. writes one flash-decoding partial (m_h, l_h, o_h) per (query lane, range); the last
//      range CTA of each query lane merges them (ticket), as the per-lane kernel does.
// Values are read once per KV lane instead of once per query head, and dequantised once.
#include "common.cuh"

namespace kvt {

constexpr int GQ_WARPS = 4;
constexpr int GQ_THREADS = GQ_WARPS * 32;
constexpr int GQ_S = 6;              // ring slots per warp (16 rows x 80 B each)
constexpr int GQ_ROWB = 80;          // INT4 record bytes at d = 128
constexpr int GQ_SLOT = 16 * GQ_ROWB;
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

template <int GQ>  // heads per KV lane (2 or 4)
__global__ void __launch_bounds__(GQ_THREADS, 3) attn_gqa_i4_kernel(
    const unsigned char* __restrict__ values, int64_t lane_stride_b, int64_t n_q, const int32_t* __restrict__ sel_tok,
    const double* __restrict__ sel_score, const int32_t* __restrict__ n_sel, int64_t sel_stride, int R, int splits,
    double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out, double* __restrict__ out64,
    double scale) {
    pdl_entry();
    constexpr int d = 128;
    constexpr int W = GQ_WIN;
    constexpr int NW = W / 32;
    constexpr int SCAN = 4;  // 32-entry batches loaded per scan step (memory-level parallelism)
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char* ring = smem;                                                   // [warps][S][16 x 80 B]
    float* wtab = reinterpret_cast<float*>(smem + GQ_WARPS * GQ_S * GQ_SLOT);     // [W][GQ] weights
    uint32_t* bm = reinterpret_cast<uint32_t*>(wtab + (size_t)W * GQ);            // [GQ][NW] head bitmaps
    uint32_t* ubm = bm + GQ * NW;                                                 // [NW] union bitmap
    int* upre = reinterpret_cast<int*>(ubm + NW);                                 // [NW] slot prefix
    uint16_t* utok = reinterpret_cast<uint16_t*>(upre + NW);                      // [W] union token offsets
    __shared__ double s_m[GQ];      // running max score per head
    __shared__ float s_rs[GQ];      // this window's rescale of the running sums
    __shared__ float s_l[GQ];       // running softmax denominators
    __shared__ int s_cur[GQ], s_end[GQ], s_wend[GQ];
    __shared__ double s_wm[GQ];
    __shared__ int s_ucnt;
    __shared__ int scan_sh[33];
    __shared__ float s_o[GQ_WARPS][GQ][d];
    __shared__ float s_om[GQ_WARPS][GQ][4];
    __shared__ int s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t kv = blockIdx.y;
    const int rg = blockIdx.x;
    const int T0 = rg * R, T1 = T0 + R;
    const double sl2 = scale * 1.4426950408889634;
    const int gid = lane >> 2, tig = lane & 3;
    const int hA = gid >> 1;             // head of A row gid (rows 8..15 stay zero)
    const bool lo_part = gid & 1;
    const unsigned char* vbase = values + kv * lane_stride_b;
    unsigned char* wring = ring + (size_t)warp * GQ_S * GQ_SLOT;
    const uint32_t wring_a = (uint32_t)__cvta_generic_to_shared(wring);

    // ---- the range's entries of every head: [lower_bound(T0), lower_bound(T1)) ----
    for (int h = warp; h < GQ; h += GQ_WARPS) {
        const int64_t li = kv * GQ + h;
        const int n = n_sel[li];
        const int32_t* tk = sel_tok + li * sel_stride;
        const int a = warp_lower_bound(tk, n, T0, lane);
        const int b = warp_lower_bound(tk, n, T1, lane);
        if (lane == 0) { s_cur[h] = a; s_end[h] = b; s_m[h] = -INFINITY; s_l[h] = 0.f; }
    }
    __syncthreads();

    float D[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) D[j][0] = D[j][1] = D[j][2] = D[j][3] = 0.f;
    float om[4] = {0.f, 0.f, 0.f, 0.f};  // sum_t w_h(t) m_t,G for head gid/2 (hi-part rows)

    for (int Tw = T0; Tw < T1; Tw += W) {
        bool any = false;
#pragma unroll
        for (int h = 0; h < GQ; ++h) any |= s_cur[h] < s_end[h];
        if (!any) break;  // block-uniform: the range's remaining windows are empty
        // ---- 1. per-head bitmaps of the window's entries + the window max ----
        for (int i = tid; i < GQ * NW; i += GQ_THREADS) bm[i] = 0u;
        __syncthreads();
        for (int h = warp; h < GQ; h += GQ_WARPS) {
            const int64_t li = kv * GQ + h;
            const int32_t* tk = sel_tok + li * sel_stride;
            const double* sc = sel_score + li * sel_stride;
            const int end = s_end[h], lim = Tw + W;
            int j = s_cur[h];
            double mx = -INFINITY;
            for (;;) {  // entries are ascending: the window's are a prefix of [j, end)
                int t[SCAN];
                double v[SCAN];
#pragma unroll
                for (int u = 0; u < SCAN; ++u) {  // ids and scores issued together: one latency
                    const int pos = j + 32 * u + lane;
                    t[u] = pos < end ? tk[pos] : INT_MAX;
                    v[u] = pos < end ? sc[pos] : -INFINITY;
                }
                int taken = 0;
#pragma unroll
                for (int u = 0; u < SCAN; ++u) {
                    const bool in = t[u] < lim;
                    taken += __popc(__ballot_sync(KVT_FULL, in));
                    if (in) {
                        const int o = t[u] - Tw;
                        atomicOr(&bm[h * NW + (o >> 5)], 1u << (o & 31));
                        mx = fmax(mx, v[u]);
                    }
                }
                j += taken;
                if (taken < 32 * SCAN) break;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(KVT_FULL, mx, off));
            if (lane == 0) {
                s_wend[h] = j;
                const double mo = s_m[h], mn = fmax(mo, mx);
                s_rs[h] = (mo == -INFINITY || mn == -INFINITY) ? 0.f : exp2f((float)((mo - mn) * sl2));
                s_wm[h] = mn;
            }
        }
        __syncthreads();
        // ---- 2. union slots (popcount prefix), token offsets, weight table ----
        for (int w = tid; w < NW; w += GQ_THREADS) {
            uint32_t u = 0;
#pragma unroll
            for (int h = 0; h < GQ; ++h) u |= bm[h * NW + w];
            ubm[w] = u;
        }
        __syncthreads();
        {
            int tot;
            const int v = tid < NW ? __popc(ubm[tid]) : 0;
            const int ex = block_excl_scan<int>(v, scan_sh, tot);
            if (tid < NW) upre[tid] = ex;
            if (tid == 0) s_ucnt = tot;
        }
        __syncthreads();
        const int ucnt = s_ucnt;
        for (int w = tid; w < NW; w += GQ_THREADS) {
            uint32_t x = ubm[w];
            int sl = upre[w];
            while (x) {
                const int bit = __ffs(x) - 1;
                x &= x - 1;
                utok[sl++] = (uint16_t)(w * 32 + bit);
            }
        }
        for (int i = tid; i < ucnt * GQ; i += GQ_THREADS) wtab[i] = 0.f;
        __syncthreads();
        for (int h = warp; h < GQ; h += GQ_WARPS) {
            const int64_t li = kv * GQ + h;
            const int32_t* tk = sel_tok + li * sel_stride;
            const double* sc = sel_score + li * sel_stride;
            const double mh = s_wm[h];
            float lsum = 0.f;
            for (int j = s_cur[h] + lane; j < s_wend[h]; j += 32) {
                const int t = tk[j] - Tw;
                const int w = t >> 5;
                const int slot = upre[w] + __popc(ubm[w] & ((1u << (t & 31)) - 1u));
                const float wt = exp2f((float)((sc[j] - mh) * sl2));
                wtab[slot * GQ + h] = wt;
                lsum += wt;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) lsum += __shfl_xor_sync(KVT_FULL, lsum, off);
            if (lane == 0) {
                s_l[h] = s_l[h] * s_rs[h] + lsum;
                s_m[h] = mh;
                s_cur[h] = s_wend[h];
            }
        }
        // running sums of this thread's head rescaled to the new max (flash decoding)
        {
            const float rs = hA < GQ ? s_rs[hA] : 0.f;
#pragma unroll
            for (int j = 0; j < 16; ++j) { D[j][0] *= rs; D[j][1] *= rs; }
#pragma unroll
            for (int G = 0; G < 4; ++G) om[G] *= rs;
        }

        // ---- 3. union rows through the per-warp ring, P.V on the tensor cores ----
        const int ntile = (ucnt + 15) / 16;
        const int my_tiles = ntile > warp ? (ntile - warp + GQ_WARPS - 1) / GQ_WARPS : 0;  // tiles w, w + 4, ...
        auto issue = [&](int it) {  // it-th tile of this warp -> ring slot it % S
            const int tile = warp + it * GQ_WARPS;
            const uint32_t dst = wring_a + (it % GQ_S) * GQ_SLOT;
#pragma unroll
            for (int p0 = 0; p0 < 96; p0 += 32) {
                const int p = p0 + lane;
                if (p < 80) {
                    const int r = p / 5, pc = p % 5;
                    int u = tile * 16 + r;
                    u = u < ucnt ? u : ucnt - 1;  // pad rows: a valid record, weight 0
                    const int t = Tw + (int)utok[u];
                    gq_cp16(dst + r * GQ_ROWB + pc * 16, vbase + (int64_t)t * GQ_ROWB + pc * 16);
                }
            }
        };
#pragma unroll
        for (int j = 0; j < GQ_S - 1; ++j) {
            if (j < my_tiles) issue(j);
            gq_commit();
        }
        __syncthreads();  // weight table complete
        for (int it = 0; it < my_tiles; ++it) {
            if (it + GQ_S - 1 < my_tiles) issue(it + GQ_S - 1);
            gq_commit();
            gq_wait<GQ_S - 1>();
            __syncwarp();
            const unsigned char* slot = wring + (it % GQ_S) * GQ_SLOT;
            const int tile = warp + it * GQ_WARPS;
            const int r0 = 2 * tig, r1 = 2 * tig + 1, r8 = 2 * tig + 8, r9 = 2 * tig + 9;
            const int u0 = tile * 16;
            auto wt = [&](int r, int h) -> float {
                const int u = u0 + r;
                return (h < GQ && u < ucnt) ? wtab[u * GQ + h] : 0.f;
            };
            const float wA0 = wt(r0, hA), wA1 = wt(r1, hA), wA8 = wt(r8, hA), wA9 = wt(r9, hA);
#pragma unroll
            for (int G = 0; G < 4; ++G) {
                // (scale, min) of the 4 rows this thread feeds
                const __half2 p0 = *reinterpret_cast<const __half2*>(slot + r0 * GQ_ROWB + 64 + 4 * G);
                const __half2 p1 = *reinterpret_cast<const __half2*>(slot + r1 * GQ_ROWB + 64 + 4 * G);
                const __half2 p8 = *reinterpret_cast<const __half2*>(slot + r8 * GQ_ROWB + 64 + 4 * G);
                const __half2 p9 = *reinterpret_cast<const __half2*>(slot + r9 * GQ_ROWB + 64 + 4 * G);
                const float s0 = __low2float(p0), s1 = __low2float(p1), s8 = __low2float(p8), s9 = __low2float(p9);
                if (!lo_part)
                    om[G] += wA0 * __high2float(p0) + wA1 * __high2float(p1) + wA8 * __high2float(p8) +
                             wA9 * __high2float(p9);
                // A = w s 2^12 as f16 (hi rows) or its f16 remainder (lo rows)
                auto split = [&](float v) -> __half {
                    const __half hi = __float2half_rn(v);
                    return lo_part ? __float2half_rn(v - __half2float(hi)) : hi;
                };
                const uint32_t a0 = pack_h2(split(wA0 * s0 * GQ_ASCALE), split(wA1 * s1 * GQ_ASCALE));
                const uint32_t a2 = pack_h2(split(wA8 * s8 * GQ_ASCALE), split(wA9 * s9 * GQ_ASCALE));
                // B: codes of word 4G + gid/2 of rows (r0, r1) and (r8, r9); bytes 0-1 (dims +0..3)
                // or 2-3 (dims +4..7) of the word by gid parity; nibble q -> dim + q
                const int wo = 4 * (4 * G + (gid >> 1));
                const uint32_t c0 = *reinterpret_cast<const uint32_t*>(slot + r0 * GQ_ROWB + wo);
                const uint32_t c1 = *reinterpret_cast<const uint32_t*>(slot + r1 * GQ_ROWB + wo);
                const uint32_t c8 = *reinterpret_cast<const uint32_t*>(slot + r8 * GQ_ROWB + wo);
                const uint32_t c9 = *reinterpret_cast<const uint32_t*>(slot + r9 * GQ_ROWB + wo);
                const uint32_t sel = (gid & 1) ? 0x7632u : 0x5410u;
                const uint32_t x01 = __byte_perm(c0, c1, sel), x89 = __byte_perm(c8, c9, sel);
                const __half2 k1024 = __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400));
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t e01 = ((x01 >> (4 * q)) & 0x000f000fu) | 0x64006400u;
                    const uint32_t e89 = ((x89 >> (4 * q)) & 0x000f000fu) | 0x64006400u;
                    const __half2 h01 = __hsub2(*reinterpret_cast<const __half2*>(&e01), k1024);
                    const __half2 h89 = __hsub2(*reinterpret_cast<const __half2*>(&e89), k1024);
                    mma_f16(D[4 * G + q], a0, 0u, a2, 0u, *reinterpret_cast<const uint32_t*>(&h01),
                            *reinterpret_cast<const uint32_t*>(&h89));
                }
            }
            __syncwarp();
        }
        gq_wait<0>();
        __syncthreads();  // ring, table and bitmaps are reused by the next window
    }

    // ---- 4. per-warp head outputs -> shared, combine warps, partials ----
    // D[4G+q][0/1]: row gid (head gid/2, hi or lo part), dims 32G + 8 tig + q and + 4 + q
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) D[j][e] += __shfl_xor_sync(KVT_FULL, D[j][e], 4);  // hi + lo rows
#pragma unroll
    for (int G = 0; G < 4; ++G) {
        float v = om[G];
        v += __shfl_xor_sync(KVT_FULL, v, 1);
        v += __shfl_xor_sync(KVT_FULL, v, 2);
        om[G] = v;
    }
    if (!lo_part && hA < GQ) {
        const float inv = 1.f / GQ_ASCALE;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int dA = 32 * (j >> 2) + 8 * tig + (j & 3);
            s_o[warp][hA][dA] = D[j][0] * inv;
            s_o[warp][hA][dA + 4] = D[j][1] * inv;
        }
        if (tig == 0)
#pragma unroll
            for (int G = 0; G < 4; ++G) s_om[warp][hA][G] = om[G];
    }
    __syncthreads();
    for (int h = 0; h < GQ; ++h) {
        const int64_t li = kv * GQ + h;
        double* P = part + (li * splits + rg) * (int64_t)(d + 2);
        for (int j = tid; j < d; j += GQ_THREADS) {
            float acc = 0.f;
#pragma unroll
            for (int w = 0; w < GQ_WARPS; ++w) acc += s_o[w][h][j] + s_om[w][h][j >> 5];
            P[2 + j] = (double)acc;
        }
        if (tid == 0) {
            P[0] = s_m[h];
            P[1] = (double)s_l[h];
        }
    }
    // ---- 5. one ticket per KV lane: the last range CTA merges the group's heads ----
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned t = atomicAdd(&tickets[kv * GQ], 1u);
        s_last = (t == (unsigned)splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int h = 0; h < GQ; ++h) gq_merge(part, splits, d, kv * GQ + h, n_q, out, out64, scale);
    if (tid == 0) tickets[kv * GQ] = 0;
}

}  // namespace kvt

using namespace kvt;

// GQA INT4 attention (kv_group g in {2, 4}, d = 128): the union pass above.  Returns
// KVT_ERR_ARG when the shape is not covered (the caller then runs the per-lane kernel).
int kvt_attn_gqa_i4(const void* values, int64_t n_lanes, int64_t lane_stride_b, int d, int kvg, int64_t n_ctx,
                    const int32_t* sel_tok, const double* sel_score, const int32_t* n_sel, int64_t sel_stride,
                    double logit_scale, void* ws, float* out, double* out64, cudaStream_t st) {
    if (d != 128 || (kvg != 2 && kvg != 4) || n_lanes % kvg || n_ctx <= 0) return KVT_ERR_ARG;
    if (((uintptr_t)values % 16) || (lane_stride_b % 16)) return KVT_ERR_SHAPE;
    if (n_ctx > (int64_t)64 * 1024 * 1024) return KVT_ERR_ARG;
    // CTAs = KV lanes x ranges: about 3 waves of 3 CTAs per SM, ranges of whole windows
    const int64_t n_kv = n_lanes / kvg;
    const int64_t n_win = (n_ctx + GQ_WIN - 1) / GQ_WIN;
    int64_t want = (3LL * 3 * kvt::sm_count() + n_kv - 1) / n_kv;
    want = kvt::imax(1, kvt::imin(kvt::imin(want, 64), n_win));
    const int R = (int)(((n_win + want - 1) / want) * GQ_WIN);
    const int splits = (int)((n_ctx + R - 1) / R);
    unsigned int* tickets = (unsigned int*)ws;
    double* part = (double*)((char*)ws + (((size_t)n_lanes * 4 + 255) & ~(size_t)255)) + 2 * n_lanes;
    const int NW = GQ_WIN / 32;
    const size_t smem = (size_t)GQ_WARPS * GQ_S * GQ_SLOT + (size_t)GQ_WIN * kvg * 4 + (size_t)(kvg + 1) * NW * 4 +
                        (size_t)NW * 4 + (size_t)GQ_WIN * 2;
#define KVT_GQ(GG)                                                                                                  \
    do {                                                                                                            \
        KVT_PER_DEVICE(size_t, configured);                                                                         \
        if (smem > configured) {                                                                                    \
            cudaError_t e = cudaFuncSetAttribute(attn_gqa_i4_kernel<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                 (int)smem);                                                        \
            if (e != cudaSuccess) return kvt_set_cuda_error(e);                                                     \
            configured = smem;                                                                                      \
        }                                                                                                           \
        launch_pdl(attn_gqa_i4_kernel<GG>, dim3((unsigned)splits, (unsigned)n_kv), dim3(GQ_THREADS), smem, st,     \
                   (const unsigned char*)values, lane_stride_b, n_lanes, sel_tok, sel_score, n_sel, sel_stride, R, \
                   splits, part, tickets, out, out64, logit_scale);                                                 \
    } while (0)
    if (kvg == 2) KVT_GQ(2);
    else KVT_GQ(4);
#undef KVT_GQ
    return kvt_check_launch();
}
