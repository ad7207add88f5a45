// score.cu -- K4 canonical float64 token logits (candidate tokens, or all tokens).
//
// Replaces importance.py:27-33 attention_logits (k.q / sqrt d) for the tokens the plan
// kept.  A warp scores 8 tokens per step: each lane loads its 4-dim group of the 8 rows
// (8 independent 64/128-bit loads in flight per lane; a 128-dim bf16 row is one coalesced
// 256 B warp access), runs its f64 fma chains, and a reduce-scatter butterfly
// (tree_8tok: 9 f64 shuffles per 8 tokens instead of 40) yields the canonical dot of
// token (lane>>2) on every quad.  HBM-bound: n_cand*d*s_K read, n_cand*12 B written.
#include "common.cuh"

namespace kvt {

constexpr int SCORE_THREADS = 256;

template <typename QT, typename T, int G, bool VEC, bool IMPLICIT>
__global__ void __launch_bounds__(SCORE_THREADS) score_kernel(
    const QT* __restrict__ q, const T* __restrict__ keys, int64_t lane_stride, int d,
    const int32_t* __restrict__ items, int64_t item_stride, const int32_t* __restrict__ n_items,
    int64_t n_implicit, double* __restrict__ out_score, int32_t* __restrict__ out_tok, int64_t out_stride) {
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
                os[pos0 + g8 + t] = dot / sd;
                if (ot) ot[pos0 + g8 + t] = (int32_t)(t0 + g8 + t);
            }
        }
    }
}

}  // namespace kvt

using namespace kvt;

static inline int sgroups_for(int d) { return d <= 128 ? 1 : d <= 256 ? 2 : d <= 512 ? 4 : d <= 1024 ? 8 : 0; }

template <typename QT, typename T, int G, bool VEC, bool IMPL>
static void launch_score(const void* q, const void* keys, int64_t n_lanes, int64_t lane_stride, int d,
                         const int32_t* items, int64_t item_stride, const int32_t* n_items, int64_t n_impl,
                         double* os, int32_t* ot, int64_t ostr, int blocks, cudaStream_t st) {
    dim3 grid(blocks, (unsigned)n_lanes);
    score_kernel<QT, T, G, VEC, IMPL><<<grid, SCORE_THREADS, 0, st>>>(
        (const QT*)q, (const T*)keys, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr);
}

template <typename QT, typename T, bool IMPL>
static int dispatch_score_t(const void* q, const void* keys, int64_t n_lanes, int64_t lane_stride, int d,
                            const int32_t* items, int64_t item_stride, const int32_t* n_items, int64_t n_impl,
                            double* os, int32_t* ot, int64_t ostr, int blocks, cudaStream_t st) {
    const bool vec = ((uintptr_t)keys % (4 * sizeof(T)) == 0) && d % 4 == 0 && lane_stride % 4 == 0;
    switch (sgroups_for(d)) {
#define KVT_CASE(GG)                                                                                                  \
    case GG:                                                                                                          \
        if (vec) launch_score<QT, T, GG, true, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items,  \
                                                     n_impl, os, ot, ostr, blocks, st);                                \
        else launch_score<QT, T, GG, false, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items,     \
                                                  n_impl, os, ot, ostr, blocks, st);                                   \
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
                          cudaStream_t st) {
#define KVT_K(QT, TT) \
    return dispatch_score_t<QT, TT, IMPL>(q, keys, n_lanes, lane_stride, d, items, item_stride, n_items, n_impl, os, ot, ostr, blocks, st)
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
                                 0, cand_score, cand_tok, cand_stride, blocks_per_lane, (cudaStream_t)stream);
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
                                nullptr, out_stride, blocks, (cudaStream_t)stream);
}
