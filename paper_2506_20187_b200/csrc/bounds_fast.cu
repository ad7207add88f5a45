// bounds_fast.cu -- K3 for the decode path: sound f32 chunk bounds with directed rounding.
//
// The drop-in bound_chunk / bound_chunks_batch (importance.py:108-137) return the canonical
// f64 bounds of abstract_bounds.cu.  The decoder only needs bounds that are SOUND (every
// canonical dot of the chunk lies in [L, U]) for the pruning of plan.cu; the selected set is
// decided later by exact scores, so it does not depend on how tight they are.  Here
//     U = sum_j q+_j max_j + q-_j min_j       (q+ = max(q, 0), q- = min(q, 0): exact)
//     L = sum_j q+_j min_j + q-_j max_j
// are accumulated in f32 with every fma / add rounded toward +inf (U) or -inf (L), so each
// partial sum bounds its exact value from the right side and U >= exact U >= every dot of
// the chunk (likewise L).  Abstracts are the decoder's bf16 ones, already rounded outward.
// Two dims per packed FFMA2 (fma.rp/rm.f32x2); the ring of bounds_tma_kernel (one producer
// thread bulk-copying 64 chunks' max rows + min rows per stage, 8 consumer warps x 8 chunks).
//
// A (the scoring error bound's sum |q||k| over a chunk) is replaced by one per-lane value,
// A_lane = RU(sum_j |q_j| M_j), with M the lane's max-|key| vector over all chunks (kept by
// the decoder next to the abstracts): A_lane >= every chunk's A, written for every chunk.
//
// GQA (kv_group g > 1): the work is enumerated over KV lanes; a stage's abstracts (one bulk
// copy per 64 chunks of a KV lane) serve all g query lanes of the group, so abstract bytes
// are read once per KV lane instead of once per query head (the reference replicates the KV
// head per query head, adapters.py:121-136 -- identical bounds, g x the bytes).
#include "common.cuh"

namespace kvt {

constexpr int BF_CONSUMERS = 8;
constexpr int BF_THREADS = (BF_CONSUMERS + 1) * 32;

__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2_rp(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rp.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fma2_rm(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// 4 bf16 (8 bytes) -> two packed f32 pairs (exact)
__device__ __forceinline__ void bf4_pairs(uint2 w, uint64_t& p01, uint64_t& p23) {
    p01 = pk2(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u));
    p23 = pk2(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u));
}

// Reduce-scatter of 8 per-chunk partials over the warp with directed adds: afterwards lane
// l holds chunk t = 4 b4 + 2 b3 + b2 (b_i = bit i of l), summed over all 32 lanes.
template <bool UP>
__device__ __forceinline__ float rs8(float (&p)[8], int lane) {
#pragma unroll
    for (int o = 16, h = 4; o >= 4; o >>= 1, h >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j < h) {
                const float keep = upper ? p[j + h] : p[j], send = upper ? p[j] : p[j + h];
                const float got = __shfl_xor_sync(KVT_FULL, send, o);
                p[j] = UP ? __fadd_ru(keep, got) : __fadd_rd(keep, got);
            }
        }
    }
    float v = p[0];
#pragma unroll
    for (int o = 2; o >= 1; o >>= 1) {
        const float got = __shfl_xor_sync(KVT_FULL, v, o);
        v = UP ? __fadd_ru(v, got) : __fadd_rd(v, got);
    }
    return v;
}

template <int G, bool PAIR>  // G = d / 128; PAIR: GQA with an even group, heads in pairs
__global__ void __launch_bounds__(BF_THREADS, 2) bounds_fast_kernel(
    const float* __restrict__ q, int64_t n, int C, int n_lanes, const __nv_bfloat16* __restrict__ amax,
    const __nv_bfloat16* __restrict__ amin, int64_t abs_lane_stride, const float* __restrict__ mag,
    double* __restrict__ U, double* __restrict__ L, double* __restrict__ A, int64_t bnd_stride, int stages, int kvg) {
    pdl_entry();
    constexpr int d = 128 * G;
    constexpr int tile = 2 * 64 * d * 2;  // 64 max rows then 64 min rows (bf16)
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * tile);
    uint64_t* empty = full + stages;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m = (n + C - 1) / C;
    const int64_t per_lane = (m + 63) / 64;
    const int n_kv = n_lanes / kvg;  // stages are per KV lane; kvg query lanes share each
    const int64_t total = per_lane * n_kv;
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], BF_CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t g0 = kvt::imin(total, (int64_t)blockIdx.x * per), g1 = kvt::imin(total, g0 + per);
    if (warp == BF_CONSUMERS) {
        if (lane == 0) {
            int ps = 0, pr = 0;
            int64_t li = g0 / per_lane, c0 = (g0 % per_lane) * 64;
            for (int64_t g = g0; g < g1; ++g) {
                const int64_t cnt = kvt::imin(64, m - c0);
                const int s = ps;
                if (pr > 0) mbar_wait(&empty[s], (uint32_t)((pr - 1) & 1));
                if (++ps == stages) { ps = 0; ++pr; }
                const uint32_t half = (uint32_t)(cnt * d * 2);
                mbar_arrive_expect_tx(&full[s], 2 * half);
                unsigned char* dst = smem + (size_t)s * tile;
                bulk_g2s(dst, amax + li * abs_lane_stride + c0 * d, half, &full[s]);
                bulk_g2s(dst + tile / 2, amin + li * abs_lane_stride + c0 * d, half, &full[s]);
                c0 += 64;
                if (c0 >= per_lane * 64) { c0 = 0; ++li; }
            }
        }
        return;
    }
    constexpr int KVG_MAX = 8;
    int64_t cur = -1;
    uint64_t qp[G][2], qn[G][2];
    float a_lane[KVG_MAX];
    __shared__ float s_alane[BF_CONSUMERS][KVG_MAX];  // PAIR: the heads' A_lane (registers freed)
    int cs = 0, cr = 0;
    int64_t li = g0 / per_lane, c0 = (g0 % per_lane) * 64;
    // q+ / q- of query lane ql (packed pairs) and, optionally, A_lane (RU sum |q| M)
    auto load_q = [&](int64_t ql, bool with_a) -> float {
        float aa = 0.f;
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float4 qv = *reinterpret_cast<const float4*>(q + ql * d + 4 * (lane + 32 * r));
            qp[r][0] = pk2(fmaxf(qv.x, 0.f), fmaxf(qv.y, 0.f));
            qp[r][1] = pk2(fmaxf(qv.z, 0.f), fmaxf(qv.w, 0.f));
            qn[r][0] = pk2(fminf(qv.x, 0.f), fminf(qv.y, 0.f));
            qn[r][1] = pk2(fminf(qv.z, 0.f), fminf(qv.w, 0.f));
            if (with_a) {
                const float4 mv = *reinterpret_cast<const float4*>(mag + (ql / kvg) * d + 4 * (lane + 32 * r));
                aa = __fmaf_ru(fabsf(qv.x), mv.x, aa);
                aa = __fmaf_ru(fabsf(qv.y), mv.y, aa);
                aa = __fmaf_ru(fabsf(qv.z), mv.z, aa);
                aa = __fmaf_ru(fabsf(qv.w), mv.w, aa);
            }
        }
        if (with_a) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) aa = __fadd_ru(aa, __shfl_xor_sync(KVT_FULL, aa, o));
        }
        return aa;
    };
    for (int64_t g = g0; g < g1; ++g) {
        const int64_t cnt = kvt::imin(64, m - c0);
        if (li != cur) {
            cur = li;
#pragma unroll
            for (int h = 0; h < KVG_MAX; ++h)
                if (h < kvg) {
                    if constexpr (PAIR) {
                        const float av = load_q(li * kvg + h, true);
                        if (lane == 0) s_alane[warp][h] = av;
                    } else {
                        a_lane[h] = load_q(li * kvg + h, true);
                    }
                }
            if (kvg > 1) load_q(li * kvg, false);
        }
        const int s = cs;
        mbar_wait(&full[s], (uint32_t)(cr & 1));
        if (++cs == stages) { cs = 0; ++cr; }
        const unsigned char* Mx = smem + (size_t)s * tile;
        const unsigned char* Mn = Mx + tile / 2;
        const int base = 8 * warp;
        if constexpr (PAIR) {
          if (base < cnt) {
            // GQA, heads in pairs: each abstract element is unpacked once for two heads and the
            // two heads' fma chains and reduce-scatters interleave (twice the independent work
            // per pass; same directed-rounding sums per head as the single-head loop below)
#pragma unroll 1
            for (int h = 0; h < kvg; h += 2) {
                uint64_t qpA[G][2], qnA[G][2], qpB[G][2], qnB[G][2];
#pragma unroll
                for (int r = 0; r < G; ++r) {
                    const float4 qa = *reinterpret_cast<const float4*>(q + (li * kvg + h) * d + 4 * (lane + 32 * r));
                    const float4 qb = *reinterpret_cast<const float4*>(q + (li * kvg + h + 1) * d + 4 * (lane + 32 * r));
                    qpA[r][0] = pk2(fmaxf(qa.x, 0.f), fmaxf(qa.y, 0.f)); qpA[r][1] = pk2(fmaxf(qa.z, 0.f), fmaxf(qa.w, 0.f));
                    qnA[r][0] = pk2(fminf(qa.x, 0.f), fminf(qa.y, 0.f)); qnA[r][1] = pk2(fminf(qa.z, 0.f), fminf(qa.w, 0.f));
                    qpB[r][0] = pk2(fmaxf(qb.x, 0.f), fmaxf(qb.y, 0.f)); qpB[r][1] = pk2(fmaxf(qb.z, 0.f), fmaxf(qb.w, 0.f));
                    qnB[r][0] = pk2(fminf(qb.x, 0.f), fminf(qb.y, 0.f)); qnB[r][1] = pk2(fminf(qb.z, 0.f), fminf(qb.w, 0.f));
                }
                float puA[8], plA[8], puB[8], plB[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    uint64_t uA = 0ull, lA = 0ull, uB = 0ull, lB = 0ull;
                    if (base + u < cnt) {
#pragma unroll
                        for (int r = 0; r < G; ++r) {
                            const int off = ((base + u) * d + 4 * (lane + 32 * r)) * 2;
                            uint64_t h01, h23, l01, l23;
                            bf4_pairs(*reinterpret_cast<const uint2*>(Mx + off), h01, h23);
                            bf4_pairs(*reinterpret_cast<const uint2*>(Mn + off), l01, l23);
                            uA = fma2_rp(qpA[r][0], h01, uA);
                            uB = fma2_rp(qpB[r][0], h01, uB);
                            lA = fma2_rm(qpA[r][0], l01, lA);
                            lB = fma2_rm(qpB[r][0], l01, lB);
                            uA = fma2_rp(qnA[r][0], l01, uA);
                            uB = fma2_rp(qnB[r][0], l01, uB);
                            lA = fma2_rm(qnA[r][0], h01, lA);
                            lB = fma2_rm(qnB[r][0], h01, lB);
                            uA = fma2_rp(qpA[r][1], h23, uA);
                            uB = fma2_rp(qpB[r][1], h23, uB);
                            lA = fma2_rm(qpA[r][1], l23, lA);
                            lB = fma2_rm(qpB[r][1], l23, lB);
                            uA = fma2_rp(qnA[r][1], l23, uA);
                            uB = fma2_rp(qnB[r][1], l23, uB);
                            lA = fma2_rm(qnA[r][1], h23, lA);
                            lB = fma2_rm(qnB[r][1], h23, lB);
                        }
                    }
                    float a, b;
                    upk2(uA, a, b); puA[u] = __fadd_ru(a, b);
                    upk2(lA, a, b); plA[u] = __fadd_rd(a, b);
                    upk2(uB, a, b); puB[u] = __fadd_ru(a, b);
                    upk2(lB, a, b); plB[u] = __fadd_rd(a, b);
                }
                const float uuA = rs8<true>(puA, lane), llA = rs8<false>(plA, lane);
                const float uuB = rs8<true>(puB, lane), llB = rs8<false>(plB, lane);
                const int t = 4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1);
                __syncwarp();
                const float aA = s_alane[warp][h], aB = s_alane[warp][h + 1];
                if ((lane & 3) == 0 && base + t < cnt) {
                    const int64_t c = c0 + base + t;
                    const int64_t qa = li * kvg + h;
                    U[qa * bnd_stride + c] = (double)uuA;
                    L[qa * bnd_stride + c] = (double)llA;
                    U[(qa + 1) * bnd_stride + c] = (double)uuB;
                    L[(qa + 1) * bnd_stride + c] = (double)llB;
                    if (A) {
                        A[qa * bnd_stride + c] = (double)aA;
                        A[(qa + 1) * bnd_stride + c] = (double)aB;
                    }
                }
            }
          }
        } else if (base < cnt) {
#pragma unroll 1
            for (int h = 0; h < kvg; ++h) {
                if (h > 0) load_q(li * kvg + h, false);  // L1-resident: 512 B per head
                float pu[8], pl[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    uint64_t u2 = 0ull, l2 = 0ull;
                    if (base + u < cnt) {
#pragma unroll
                        for (int r = 0; r < G; ++r) {
                            const int off = ((base + u) * d + 4 * (lane + 32 * r)) * 2;
                            uint64_t h01, h23, l01, l23;
                            bf4_pairs(*reinterpret_cast<const uint2*>(Mx + off), h01, h23);
                            bf4_pairs(*reinterpret_cast<const uint2*>(Mn + off), l01, l23);
                            u2 = fma2_rp(qp[r][0], h01, u2);
                            u2 = fma2_rp(qn[r][0], l01, u2);
                            u2 = fma2_rp(qp[r][1], h23, u2);
                            u2 = fma2_rp(qn[r][1], l23, u2);
                            l2 = fma2_rm(qp[r][0], l01, l2);
                            l2 = fma2_rm(qn[r][0], h01, l2);
                            l2 = fma2_rm(qp[r][1], l23, l2);
                            l2 = fma2_rm(qn[r][1], h23, l2);
                        }
                    }
                    float a, b;
                    upk2(u2, a, b);
                    pu[u] = __fadd_ru(a, b);
                    upk2(l2, a, b);
                    pl[u] = __fadd_rd(a, b);
                }
                const float uu = rs8<true>(pu, lane);
                const float ll = rs8<false>(pl, lane);
                const int t = 4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1);
                float ah = a_lane[0];
#pragma unroll
                for (int x = 1; x < KVG_MAX; ++x)
                    if (x == h) ah = a_lane[x];
                if ((lane & 3) == 0 && base + t < cnt) {
                    const int64_t c = c0 + base + t;
                    const int64_t ql = li * kvg + h;
                    U[ql * bnd_stride + c] = (double)uu;
                    L[ql * bnd_stride + c] = (double)ll;
                    if (A) A[ql * bnd_stride + c] = (double)ah;
                }
            }
            if (kvg > 1) load_q(li * kvg, false);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        c0 += 64;
        if (c0 >= per_lane * 64) { c0 = 0; ++li; }
    }
}

}  // namespace kvt

using namespace kvt;

extern "C" int kvt_chunk_bounds_fast(const float* q, int64_t n_lanes, int d, int64_t n, int C, const void* amax,
                                     const void* amin, int64_t abs_lane_stride, const float* mag, double* U, double* L,
                                     double* A, int64_t bnd_stride, void* stream) {
    if (!q || !amax || !amin || !mag || !U || !L || n_lanes < 0 || n < 0 || C < 1) return KVT_ERR_ARG;
    if (d != 128 && d != 256) return KVT_ERR_SHAPE;
    if (((uintptr_t)q % 16) || ((uintptr_t)mag % 16) || ((uintptr_t)amax % 16) || ((uintptr_t)amin % 16) ||
        (abs_lane_stride * 2) % 16)
        return KVT_ERR_SHAPE;
    if (n_lanes == 0 || n == 0) return KVT_OK;
    if (n_lanes > 2147483647LL) return KVT_ERR_ARG;
    if (kv_group_current() > 8 || n_lanes % kv_group_current()) return KVT_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int tile = 2 * 64 * d * 2;
    const int stages = (int)kvt::imax(2, kvt::imin(4, (100 * 1024) / tile));
    const size_t smem = (size_t)stages * tile + 16 * (size_t)stages + 16;
    static int per_sm_slots[kvt::kMaxDevices][2][3] = {};
    const int kvg = kv_group_current();
    const bool pair = kvg > 1 && (kvg & 1) == 0;
    int (&per_sm)[3] = per_sm_slots[kvt::current_device()][pair ? 1 : 0];
    const int sms = kvt::sm_count();
    const int G = d / 128;
#define KVT_BF(GG, PP)                                                                                                \
    do {                                                                                                              \
        if (!per_sm[GG]) {                                                                                            \
            cudaFuncSetAttribute(bounds_fast_kernel<GG, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            per_sm[GG] = resident_per_sm(bounds_fast_kernel<GG, PP>, BF_THREADS, smem, 1);                            \
        }                                                                                                             \
        launch_pdl(bounds_fast_kernel<GG, PP>, dim3(sms * per_sm[GG]), dim3(BF_THREADS), smem, st, q, n, C,         \
                   (int)n_lanes, (const __nv_bfloat16*)amax, (const __nv_bfloat16*)amin, abs_lane_stride, mag, U, L, \
                   A, bnd_stride, stages, kvg);                                                                       \
    } while (0)
    if (G == 1) {
        if (pair) KVT_BF(1, true);
        else KVT_BF(1, false);
    } else {
        if (pair) KVT_BF(2, true);
        else KVT_BF(2, false);
    }
#undef KVT_BF
    return kvt_check_launch();
}
