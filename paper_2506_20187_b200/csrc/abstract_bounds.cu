// abstract_bounds.cu -- K1 chunk abstracts and K3 query-vs-abstract bounds.
//
// K1 replaces importance.py:80-87 make_abstract (+ the per-leaf loop of build_partition,
// chunk_tree.py:199-208): element-wise max / min of a chunk's key rows.  One warp per
// chunk; lane l owns dims 4l..4l+3 (+128r), so a 128-dim bf16 row is one coalesced 256 B
// warp load; 8 rows are kept in flight per lane.  HBM-bound: reads C*d*s_K, writes 2*d*4.
//
// K3 replaces importance.py:108-137 bound_chunk / bound_chunks_batch: per dimension the
// query sign picks the max or min key, U = sum q*hi, L = sum q*lo, in the canonical f64
// order, widened by 2*gamma*A (A = sum |q| max(|hi|,|lo|)) so U >= every canonical token
// score in the chunk >= L.  Exact for single-row chunks and for chunks whose unwidened U == L
// (round-to-nearest fma/add are monotone, so the unwidened chains already enclose every
// canonical dot; U == L pins them all to that value).  One warp per chunk, reads the
// 2*d abstract floats once.  HBM-bound on abstract bytes (m*2*d*4 per lane).
#include <type_traits>

#include "common.cuh"

namespace kvt {

template <typename T> struct AbsOf { using type = float; };
template <> struct AbsOf<double> { using type = double; };

// Abstract stores.  bf16 abstracts (the decoder's compact form, half the bytes of f32) are
// rounded OUTWARD -- max up, min down -- so they still bound every key and the bounds stay
// sound; f32/f64 stores are exact (f32/bf16/f16 keys are exact in f32).
template <typename A> __device__ __forceinline__ void st_max(A* p, double v) { *p = (A)v; }
template <typename A> __device__ __forceinline__ void st_min(A* p, double v) { *p = (A)v; }
template <> __device__ __forceinline__ void st_max<__nv_bfloat16>(__nv_bfloat16* p, double v) {
    *p = __float2bfloat16_ru((float)v);
}
template <> __device__ __forceinline__ void st_min<__nv_bfloat16>(__nv_bfloat16* p, double v) {
    *p = __float2bfloat16_rd((float)v);
}

template <typename T, int G, bool VEC, typename A>
__global__ void __launch_bounds__(256) abstract_grid_kernel(
    const T* __restrict__ keys, int64_t lane_stride, int64_t n, int d, int C, int64_t c_begin,
    int64_t c_end, A* __restrict__ amax, A* __restrict__ amin, int64_t abs_lane_stride) {
    const int lane = threadIdx.x & 31;
    const int64_t lane_i = blockIdx.y;
    const int64_t nchunks = c_end - c_begin;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const T* base = keys + lane_i * lane_stride;
    // extrema in the key's own precision (f32 holds f32/bf16/f16 keys exactly); rows in
    // flight per lane shrink with G so the d = 512/1024 instantiations stay in registers
    using W = typename std::conditional<std::is_same<T, double>::value, double, float>::type;
    constexpr int GW = G * (int)sizeof(W) / 4;  // register words per element group
    constexpr int UR = GW <= 2 ? 8 : (GW <= 4 ? 4 : (GW <= 8 ? 2 : 1));
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nchunks; w += warps) {
        const int64_t c = c_begin + w;
        const int64_t s = c * C, e = min(n, s + C);
        W mx[G][4], mn[G][4];
#pragma unroll
        for (int r = 0; r < G; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i) { mx[r][i] = -INFINITY; mn[r][i] = INFINITY; }
        int64_t t = s;
        for (; t + UR <= e; t += UR) {
            W v[UR][G][4];
#pragma unroll
            for (int u = 0; u < UR; ++u)
#pragma unroll
                for (int r = 0; r < G; ++r) {
                    const int g = lane + 32 * r;
                    double x[4] = {0.0, 0.0, 0.0, 0.0};
                    if (4 * g < d) load_group<T, VEC>(base + (t + u) * d, g, d, x);
#pragma unroll
                    for (int i = 0; i < 4; ++i) v[u][r][i] = (W)x[i];
                }
#pragma unroll
            for (int u = 0; u < UR; ++u)
#pragma unroll
                for (int r = 0; r < G; ++r)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        mx[r][i] = max(mx[r][i], v[u][r][i]);
                        mn[r][i] = min(mn[r][i], v[u][r][i]);
                    }
        }
        for (; t < e; ++t) {
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const int g = lane + 32 * r;
                if (4 * g < d) {
                    double v[4];
                    load_group<T, VEC>(base + t * d, g, d, v);
#pragma unroll
                    for (int i = 0; i < 4; ++i) { mx[r][i] = max(mx[r][i], (W)v[i]); mn[r][i] = min(mn[r][i], (W)v[i]); }
                }
            }
        }
        A* omx = amax + lane_i * abs_lane_stride + c * d;
        A* omn = amin + lane_i * abs_lane_stride + c * d;
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const int g = lane + 32 * r;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = 4 * g + i;
                if (j < d) { st_max<A>(omx + j, mx[r][i]); st_min<A>(omn + j, mn[r][i]); }
            }
        }
    }
}

template <typename T, int G, bool VEC>
__global__ void __launch_bounds__(256) abstract_spans_kernel(
    const T* __restrict__ keys, int64_t lane_stride, int d, int64_t n_spans,
    const int32_t* __restrict__ lane_of, const int32_t* __restrict__ starts,
    const int32_t* __restrict__ ends, typename AbsOf<T>::type* __restrict__ amax,
    typename AbsOf<T>::type* __restrict__ amin) {
    using A = typename AbsOf<T>::type;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < n_spans; w += warps) {
        const T* base = keys + (int64_t)lane_of[w] * lane_stride;
        const int64_t s = starts[w], e = ends[w];
        double mx[G][4], mn[G][4];
#pragma unroll
        for (int r = 0; r < G; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i) { mx[r][i] = -INFINITY; mn[r][i] = INFINITY; }
        for (int64_t t = s; t < e; ++t) {
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const int g = lane + 32 * r;
                if (4 * g < d) {
                    double v[4];
                    load_group<T, VEC>(base + t * d, g, d, v);
#pragma unroll
                    for (int i = 0; i < 4; ++i) { mx[r][i] = fmax(mx[r][i], v[i]); mn[r][i] = fmin(mn[r][i], v[i]); }
                }
            }
        }
        A* omx = amax + w * d;
        A* omn = amin + w * d;
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const int g = lane + 32 * r;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = 4 * g + i;
                if (j < d) { omx[j] = (A)mx[r][i]; omn[j] = (A)mn[r][i]; }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// K3 bounds
// ------------------------------------------------------------------------------------------

template <typename QT, typename AT, int G>
__global__ void __launch_bounds__(256, 3) bounds_kernel(
    const QT* __restrict__ q, int d, int64_t n, int C, const int32_t* __restrict__ leaf_start,
    const int32_t* __restrict__ n_leaves, int64_t leaf_stride, const AT* __restrict__ amax,
    const AT* __restrict__ amin, int64_t abs_lane_stride, double* __restrict__ U,
    double* __restrict__ L, double* __restrict__ A, int64_t bnd_stride, int scaled) {
    // 4 chunks per warp step: 8 independent 16 B abstract loads in flight per lane, then
    // three reduce-scatter trees (U, L, A) leave chunk (lane >> 3) & 3 on each lane octet.
    // Outputs are raw (unscaled) bounds unless `scaled` (the importance.py API form).
    const int lane = threadIdx.x & 31;
    const int64_t lane_i = blockIdx.y;
    const int64_t nl = leaf_start ? (int64_t)n_leaves[lane_i] : (n + C - 1) / C;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5) * 4;
    double qr[G][4];
#pragma unroll
    for (int r = 0; r < G; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = 4 * (lane + 32 * r) + i;
            qr[r][i] = j < d ? (double)q[lane_i * d + j] : 0.0;
        }
    const double sd = sqrt((double)d);
    const double fac = slack_factor(d);
    const AT* mxb = amax + lane_i * abs_lane_stride;
    const AT* mnb = amin + lane_i * abs_lane_stride;
    const int32_t* ls = leaf_start ? leaf_start + lane_i * leaf_stride : nullptr;
    for (int64_t c0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4; c0 < nl; c0 += wstride) {
        double pu[4], pl[4], pa[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pu[u] = 0.0; pl[u] = 0.0; pa[u] = 0.0;
            const int64_t c = c0 + u;
            if (c < nl) {
                const AT* M = mxb + c * d;
                const AT* N = mnb + c * d;
#pragma unroll
                for (int r = 0; r < G; ++r) {
                    const int g = lane + 32 * r;
                    if (4 * g < d) {
                        double hv[4], lv[4];
                        if (d % 4 == 0) {
                            Elem<AT>::load4(M + 4 * g, hv);
                            Elem<AT>::load4(N + 4 * g, lv);
                        } else {
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                hv[i] = 4 * g + i < d ? (double)M[4 * g + i] : 0.0;
                                lv[i] = 4 * g + i < d ? (double)N[4 * g + i] : 0.0;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            if (4 * g + i < d) {
                                const double qj = qr[r][i];
                                const double hi = qj >= 0.0 ? hv[i] : lv[i];
                                const double lo = qj >= 0.0 ? lv[i] : hv[i];
                                pu[u] = fma(qj, hi, pu[u]);
                                pl[u] = fma(qj, lo, pl[u]);
                                pa[u] = fma(fabs(qj), fmax(fabs(hv[i]), fabs(lv[i])), pa[u]);
                            }
                        }
                    }
                }
            }
        }
        double u_ = tree_4tok(pu, lane), l_ = tree_4tok(pl, lane), a_ = tree_4tok(pa, lane);
        const int t = (lane >> 3) & 3;
        const int64_t c = c0 + t;
        if ((lane & 7) == 0 && c < nl) {
            int64_t rows;
            if (ls) rows = ((c + 1 < nl) ? (int64_t)ls[c + 1] : n) - ls[c];
            else rows = kvt::imin((int64_t)C, n - c * C);
            if (rows > 1 && u_ != l_) {  // u_ == l_: every canonical dot equals u_ (exact)
                const double slack = a_ * fac;
                u_ = u_ + slack;
                l_ = l_ - slack;
            }
            U[lane_i * bnd_stride + c] = scaled ? u_ / sd : u_;
            L[lane_i * bnd_stride + c] = scaled ? l_ / sd : l_;
            if (A) A[lane_i * bnd_stride + c] = a_;  // sum |q| max(|max|,|min|): bounds sum |q.k| in the chunk
        }
    }
}

// ------------------------------------------------------------------------------------------
// K3, TMA-staged variant for the uniform grid (the decoder's case): persistent CTAs walk the
// flattened (lane, 64-chunk block) list; one producer thread bulk-copies each block's max
// rows and min rows (contiguous, 2 x 64 x d x s_A bytes) into a shared-memory ring, eight
// consumer warps bound eight chunks each straight from shared memory.  Same arithmetic as
// bounds_kernel (canonical order, outward slack), different data movement.
// ------------------------------------------------------------------------------------------

constexpr int BT_CONSUMERS = 8;
constexpr int BT_THREADS = (BT_CONSUMERS + 1) * 32;

template <typename QT, typename AT, int G>
__global__ void __launch_bounds__(BT_THREADS, 2) bounds_tma_kernel(
    const QT* __restrict__ q, int d, int64_t n, int C, int n_lanes, const AT* __restrict__ amax,
    const AT* __restrict__ amin, int64_t abs_lane_stride, double* __restrict__ U, double* __restrict__ L,
    double* __restrict__ A, int64_t bnd_stride, int scaled, int stages) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tile = 2 * 64 * d * (int)sizeof(AT);  // max rows then min rows
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * tile);
    uint64_t* empty = full + stages;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m = (n + C - 1) / C;
    const int64_t per_lane = (m + 63) / 64;
    const int64_t total = per_lane * n_lanes;
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], BT_CONSUMERS); }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t g0 = kvt::imin(total, (int64_t)blockIdx.x * per), g1 = kvt::imin(total, g0 + per);
    if (warp == BT_CONSUMERS) {
        if (lane == 0) {
            int64_t i = 0;
            int ps = 0, pr = 0;
            for (int64_t g = g0; g < g1; ++g, ++i) {
                const int64_t li = g / per_lane, c0 = (g % per_lane) * 64;
                const int64_t cnt = kvt::imin(64, m - c0);
                // ring position without integer division: stage ps, fill round pr
                const int s = ps;
                if (pr > 0) mbar_wait(&empty[s], (uint32_t)((pr - 1) & 1));
                if (++ps == stages) { ps = 0; ++pr; }
                const uint32_t half = (uint32_t)(cnt * d * sizeof(AT));
                mbar_arrive_expect_tx(&full[s], 2 * half);
                unsigned char* dst = smem + (size_t)s * tile;
                bulk_g2s(dst, amax + li * abs_lane_stride + c0 * d, half, &full[s]);
                bulk_g2s(dst + tile / 2, amin + li * abs_lane_stride + c0 * d, half, &full[s]);
            }
        }
        return;
    }
    const double sd = sqrt((double)d);
    const double fac = slack_factor(d);
    int64_t cur = -1;
    double qr[G][4];
    int64_t i = 0;
    int cs = 0, cr = 0;
    for (int64_t g = g0; g < g1; ++g, ++i) {
        const int64_t li = g / per_lane, c0 = (g % per_lane) * 64;
        const int64_t cnt = kvt::imin(64, m - c0);
        if (li != cur) {
            cur = li;
#pragma unroll
            for (int r = 0; r < G; ++r)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = 4 * (lane + 32 * r) + e;
                    qr[r][e] = j < d ? (double)q[li * d + j] : 0.0;
                }
        }
        const int s = cs;
        mbar_wait(&full[s], (uint32_t)(cr & 1));
        if (++cs == stages) { cs = 0; ++cr; }
        const AT* Mx = reinterpret_cast<const AT*>(smem + (size_t)s * tile);
        const AT* Mn = Mx + 64 * d;
        const int base = 8 * warp;
        if (base < cnt) {
            double pu[8], pl[8], pa[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                pu[u] = 0.0; pl[u] = 0.0; pa[u] = 0.0;
                if (base + u < cnt) {
#pragma unroll
                    for (int r = 0; r < G; ++r) {
                        double hv[4], lv[4];
                        lds4<AT>(Mx + (int64_t)(base + u) * d + 4 * (lane + 32 * r), hv);
                        lds4<AT>(Mn + (int64_t)(base + u) * d + 4 * (lane + 32 * r), lv);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const double qj = qr[r][e];
                            const double hi = qj >= 0.0 ? hv[e] : lv[e];
                            const double lo = qj >= 0.0 ? lv[e] : hv[e];
                            pu[u] = fma(qj, hi, pu[u]);
                            pl[u] = fma(qj, lo, pl[u]);
                            pa[u] = fma(fabs(qj), fmax(fabs(hv[e]), fabs(lv[e])), pa[u]);
                        }
                    }
                }
            }
            double u_ = tree_8tok<double>(pu, lane), l_ = tree_8tok<double>(pl, lane), a_ = tree_8tok<double>(pa, lane);
            const int t = (lane >> 2) & 7;
            const int64_t c = c0 + base + t;
            if ((lane & 3) == 0 && base + t < cnt) {
                const int64_t rows = kvt::imin((int64_t)C, n - c * C);
                if (rows > 1 && u_ != l_) {  // degenerate chunk (max == min): exact
                    const double slack = a_ * fac;
                    u_ = u_ + slack;
                    l_ = l_ - slack;
                }
                U[li * bnd_stride + c] = scaled ? u_ / sd : u_;
                L[li * bnd_stride + c] = scaled ? l_ / sd : l_;
                if (A) A[li * bnd_stride + c] = a_;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

}  // namespace kvt

using namespace kvt;

static inline int groups_for(int d) { return d <= 128 ? 1 : d <= 256 ? 2 : d <= 512 ? 4 : d <= 1024 ? 8 : 0; }

static inline bool aligned16(const void* p, int64_t elem_bytes, int64_t lane_stride, int d) {
    return ((uintptr_t)p % (4 * elem_bytes) == 0) && (d % 4 == 0) && (lane_stride % 4 == 0);
}

template <typename T, int G, bool VEC>
static void launch_abs_grid(const void* keys, int64_t n_lanes, int64_t lane_stride, int64_t n, int d, int C,
                            int64_t cb, int64_t ce, void* amax, void* amin, int64_t als, bool bf16_abs,
                            cudaStream_t st) {
    using A = typename AbsOf<T>::type;
    const int64_t nch = ce - cb;
    int gx = (int)kvt::imin((nch + 7) / 8, 4096);
    if (gx < 1) gx = 1;
    dim3 grid(gx, (unsigned)n_lanes);
    if (bf16_abs)
        abstract_grid_kernel<T, G, VEC, __nv_bfloat16><<<grid, 256, 0, st>>>(
            (const T*)keys, lane_stride, n, d, C, cb, ce, (__nv_bfloat16*)amax, (__nv_bfloat16*)amin, als);
    else
        abstract_grid_kernel<T, G, VEC, A><<<grid, 256, 0, st>>>((const T*)keys, lane_stride, n, d, C, cb, ce,
                                                                 (A*)amax, (A*)amin, als);
}

template <typename T>
static int dispatch_abs_grid(const void* keys, int64_t n_lanes, int64_t lane_stride, int64_t n, int d, int C,
                             int64_t cb, int64_t ce, void* amax, void* amin, int64_t als, bool bf, cudaStream_t st) {
    const bool vec = aligned16(keys, sizeof(T), lane_stride, d);
    switch (groups_for(d)) {
#define KVT_CASE(GG)                                                                                        \
    case GG:                                                                                                \
        if (vec) launch_abs_grid<T, GG, true>(keys, n_lanes, lane_stride, n, d, C, cb, ce, amax, amin, als, bf, st); \
        else launch_abs_grid<T, GG, false>(keys, n_lanes, lane_stride, n, d, C, cb, ce, amax, amin, als, bf, st);   \
        break;
        KVT_CASE(1) KVT_CASE(2) KVT_CASE(4) KVT_CASE(8)
#undef KVT_CASE
        default: return KVT_ERR_SHAPE;
    }
    return kvt_check_launch();
}

extern "C" int kvt_abstract_build(const void* keys, int key_dtype, int64_t n_lanes, int64_t lane_stride, int64_t n,
                                  int d, int C, int64_t c_begin, int64_t c_end, void* amax, void* amin,
                                  int abs_dtype, int64_t abs_lane_stride, void* stream) {
    if (!keys || !amax || !amin || n_lanes < 0 || n < 0 || d < 1 || C < 1) return KVT_ERR_ARG;
    if (c_begin < 0 || c_end < c_begin || c_end > (n + C - 1) / C) return KVT_ERR_SHAPE;
    if (n_lanes == 0 || c_end == c_begin) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const bool bf = abs_dtype == KVT_BF16;
    const int natural = key_dtype == KVT_F64 ? KVT_F64 : KVT_F32;
    if (!bf && abs_dtype != natural) return KVT_ERR_DTYPE;
    switch (key_dtype) {
        case KVT_I4: return kvt_abstract_build_i4(keys, n_lanes, lane_stride, n, d, C, c_begin, c_end, amax, amin, abs_lane_stride, bf, st);
        case KVT_F32: return dispatch_abs_grid<float>(keys, n_lanes, lane_stride, n, d, C, c_begin, c_end, amax, amin, abs_lane_stride, bf, st);
        case KVT_F64: return dispatch_abs_grid<double>(keys, n_lanes, lane_stride, n, d, C, c_begin, c_end, amax, amin, abs_lane_stride, bf, st);
        case KVT_BF16: return dispatch_abs_grid<__nv_bfloat16>(keys, n_lanes, lane_stride, n, d, C, c_begin, c_end, amax, amin, abs_lane_stride, bf, st);
        case KVT_F16: return dispatch_abs_grid<__half>(keys, n_lanes, lane_stride, n, d, C, c_begin, c_end, amax, amin, abs_lane_stride, bf, st);
        default: return KVT_ERR_DTYPE;
    }
}

template <typename T, int G, bool VEC>
static void launch_abs_spans(const void* keys, int64_t lane_stride, int d, int64_t ns, const int32_t* lane_of,
                             const int32_t* s, const int32_t* e, void* amax, void* amin, cudaStream_t st) {
    using A = typename AbsOf<T>::type;
    int gx = (int)kvt::imin((ns + 7) / 8, 8192);
    abstract_spans_kernel<T, G, VEC><<<gx, 256, 0, st>>>((const T*)keys, lane_stride, d, ns, lane_of, s, e,
                                                         (A*)amax, (A*)amin);
}

template <typename T>
static int dispatch_abs_spans(const void* keys, int64_t lane_stride, int d, int64_t ns, const int32_t* lane_of,
                              const int32_t* s, const int32_t* e, void* amax, void* amin, cudaStream_t st) {
    const bool vec = aligned16(keys, sizeof(T), lane_stride, d);
    switch (groups_for(d)) {
#define KVT_CASE(GG)                                                                                  \
    case GG:                                                                                          \
        if (vec) launch_abs_spans<T, GG, true>(keys, lane_stride, d, ns, lane_of, s, e, amax, amin, st); \
        else launch_abs_spans<T, GG, false>(keys, lane_stride, d, ns, lane_of, s, e, amax, amin, st);    \
        break;
        KVT_CASE(1) KVT_CASE(2) KVT_CASE(4) KVT_CASE(8)
#undef KVT_CASE
        default: return KVT_ERR_SHAPE;
    }
    return kvt_check_launch();
}

extern "C" int kvt_abstract_spans(const void* keys, int key_dtype, int64_t lane_stride, int d, int64_t n_spans,
                                  const int32_t* lane_of, const int32_t* starts, const int32_t* ends, void* amax,
                                  void* amin, void* stream) {
    if (!keys || !lane_of || !starts || !ends || !amax || !amin || d < 1 || n_spans < 0) return KVT_ERR_ARG;
    if (n_spans == 0) return KVT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    switch (key_dtype) {
        case KVT_F32: return dispatch_abs_spans<float>(keys, lane_stride, d, n_spans, lane_of, starts, ends, amax, amin, st);
        case KVT_F64: return dispatch_abs_spans<double>(keys, lane_stride, d, n_spans, lane_of, starts, ends, amax, amin, st);
        case KVT_BF16: return dispatch_abs_spans<__nv_bfloat16>(keys, lane_stride, d, n_spans, lane_of, starts, ends, amax, amin, st);
        case KVT_F16: return dispatch_abs_spans<__half>(keys, lane_stride, d, n_spans, lane_of, starts, ends, amax, amin, st);
        default: return KVT_ERR_DTYPE;
    }
}

template <typename QT, typename AT, int G>
static void launch_bounds(const void* q, int64_t n_lanes, int d, int64_t n, int C, const int32_t* ls,
                          const int32_t* nl, int64_t lstr, const void* amax, const void* amin, int64_t als,
                          double* U, double* L, double* A, int64_t bs, int64_t max_leaves, int scaled, cudaStream_t st) {
    // uniform grid, vector-aligned rows, d = 128 G: the TMA-staged kernel
    const int64_t row = (int64_t)d * sizeof(AT);
    if (!ls && sizeof(AT) <= 4 && d == 128 * G && G <= 2 && row % 16 == 0 && ((uintptr_t)amax % 16) == 0 && ((uintptr_t)amin % 16) == 0 &&
        (als * (int64_t)sizeof(AT)) % 16 == 0 && n_lanes <= 2147483647LL && 2 * (2 * 64 * row) <= 200 * 1024) {
        const int tile = (int)(2 * 64 * row);
        const int stages = (int)kvt::imax(2, kvt::imin(4, (100 * 1024) / tile));
        const size_t smem = (size_t)stages * tile + 16 * (size_t)stages + 16;
        KVT_PER_DEVICE(bool, configured);
        if (!configured) {
            cudaFuncSetAttribute(bounds_tma_kernel<QT, AT, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            configured = true;
        }
        bounds_tma_kernel<QT, AT, G><<<kvt::sm_count() * (smem <= 110 * 1024 ? 2 : 1), BT_THREADS, smem, st>>>(
            (const QT*)q, d, n, C, (int)n_lanes, (const AT*)amax, (const AT*)amin, als, U, L, A, bs, scaled, stages);
        return;
    }
    int gx = (int)kvt::imax(1, kvt::imin((max_leaves + 31) / 32, 1024));
    // keep ~8 CTAs per SM in total when lanes are few
    dim3 grid(gx, (unsigned)n_lanes);
    bounds_kernel<QT, AT, G><<<grid, 256, 0, st>>>((const QT*)q, d, n, C, ls, nl, lstr, (const AT*)amax,
                                                   (const AT*)amin, als, U, L, A, bs, scaled);
}

template <typename QT, typename AT>
static int dispatch_bounds(const void* q, int64_t n_lanes, int d, int64_t n, int C, const int32_t* ls,
                           const int32_t* nl, int64_t lstr, const void* amax, const void* amin, int64_t als,
                           double* U, double* L, double* A, int64_t bs, int64_t max_leaves, int scaled, cudaStream_t st) {
    switch (groups_for(d)) {
#define KVT_CASE(GG) \
    case GG: launch_bounds<QT, AT, GG>(q, n_lanes, d, n, C, ls, nl, lstr, amax, amin, als, U, L, A, bs, max_leaves, scaled, st); break;
        KVT_CASE(1) KVT_CASE(2) KVT_CASE(4) KVT_CASE(8)
#undef KVT_CASE
        default: return KVT_ERR_SHAPE;
    }
    return kvt_check_launch();
}

extern "C" int kvt_chunk_bounds(const void* q, int q_dtype, int64_t n_lanes, int d, int64_t n, int C,
                                const int32_t* leaf_start, const int32_t* n_leaves, int64_t leaf_stride,
                                const void* amax, const void* amin, int abs_dtype, int64_t abs_lane_stride, double* U,
                                double* L, double* A, int64_t bnd_stride, int scaled, void* stream) {
    if (!q || !amax || !amin || !U || !L || d < 1 || n < 0 || n_lanes < 0) return KVT_ERR_ARG;
    if (!leaf_start && C < 1) return KVT_ERR_ARG;
    if (leaf_start && !n_leaves) return KVT_ERR_ARG;
    if (n_lanes == 0 || n == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    const int64_t max_leaves = leaf_start ? leaf_stride : (n + C - 1) / C;
    cudaStream_t st = (cudaStream_t)stream;
    if (q_dtype == KVT_F32 && abs_dtype == KVT_F32)
        return dispatch_bounds<float, float>(q, n_lanes, d, n, C, leaf_start, n_leaves, leaf_stride, amax, amin, abs_lane_stride, U, L, A, bnd_stride, max_leaves, scaled, st);
    if (q_dtype == KVT_F64 && abs_dtype == KVT_F32)
        return dispatch_bounds<double, float>(q, n_lanes, d, n, C, leaf_start, n_leaves, leaf_stride, amax, amin, abs_lane_stride, U, L, A, bnd_stride, max_leaves, scaled, st);
    if (q_dtype == KVT_F32 && abs_dtype == KVT_F64)
        return dispatch_bounds<float, double>(q, n_lanes, d, n, C, leaf_start, n_leaves, leaf_stride, amax, amin, abs_lane_stride, U, L, A, bnd_stride, max_leaves, scaled, st);
    if (q_dtype == KVT_F32 && abs_dtype == KVT_BF16)
        return dispatch_bounds<float, __nv_bfloat16>(q, n_lanes, d, n, C, leaf_start, n_leaves, leaf_stride, amax, amin, abs_lane_stride, U, L, A, bnd_stride, max_leaves, scaled, st);
    if (q_dtype == KVT_F64 && abs_dtype == KVT_BF16)
        return dispatch_bounds<double, __nv_bfloat16>(q, n_lanes, d, n, C, leaf_start, n_leaves, leaf_stride, amax, amin, abs_lane_stride, U, L, A, bnd_stride, max_leaves, scaled, st);
    if (q_dtype == KVT_F64 && abs_dtype == KVT_F64)
        return dispatch_bounds<double, double>(q, n_lanes, d, n, C, leaf_start, n_leaves, leaf_stride, amax, amin, abs_lane_stride, U, L, A, bnd_stride, max_leaves, scaled, st);
    return KVT_ERR_DTYPE;
}

// ------------------------------------------------------------------------------------------
// K2: merge_abstracts (importance.py:90-100) over segments of consecutive chunk abstracts --
// the union abstract of a desert run (merge_desert, chunk_tree.py:344-379), of the pieces of
// a rebuilt leaf, or of f fine chunks (a coarser grid built from a finer one without
// re-reading the keys).  Element-wise max / min are exact in every dtype, so the result is
// bit-identical to folding merge_abstracts pairwise (and, for outward-rounded bf16
// abstracts, to building the coarse grid from the keys: rounding up is monotone).  One warp
// per segment; lane l owns dims 4l..4l+3 (+128r).
// ------------------------------------------------------------------------------------------
namespace kvt {

template <typename T>
__global__ void __launch_bounds__(256) abstract_merge_kernel(
    const T* __restrict__ amax, const T* __restrict__ amin, int64_t in_lane_stride, int d, int64_t n_seg,
    const int32_t* __restrict__ seg_lane, const int32_t* __restrict__ seg_begin, const int32_t* __restrict__ seg_end,
    int factor, int64_t m_in, int64_t m_out, T* __restrict__ omax, T* __restrict__ omin, int64_t out_lane_stride) {
    using W = typename std::conditional<std::is_same<T, double>::value, double, float>::type;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < n_seg; s += warps) {
        int64_t ln, b, e, orow;
        if (seg_lane) {  // explicit segments: output row s
            ln = seg_lane[s];
            b = seg_begin[s];
            e = seg_end[s];
            orow = s * d;
        } else {  // uniform coarsening: segment (lane, j) = fine chunks [j f, (j + 1) f)
            ln = s / m_out;
            const int64_t j = s % m_out;
            b = j * factor;
            e = kvt::imin(m_in, b + factor);
            orow = ln * out_lane_stride + j * d;
        }
        const T* pmx = amax + ln * in_lane_stride;
        const T* pmn = amin + ln * in_lane_stride;
        for (int g = lane; 4 * g < d; g += 32) {
            W mx[4], mn[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { mx[i] = -INFINITY; mn[i] = INFINITY; }
            for (int64_t c = b; c < e; ++c) {
                double x[4], y[4];
                load_group<T, false>(pmx + c * d, g, d, x);
                load_group<T, false>(pmn + c * d, g, d, y);
#pragma unroll
                for (int i = 0; i < 4; ++i) { mx[i] = max(mx[i], (W)x[i]); mn[i] = min(mn[i], (W)y[i]); }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (4 * g + i < d && e > b) { omax[orow + 4 * g + i] = (T)mx[i]; omin[orow + 4 * g + i] = (T)mn[i]; }
        }
    }
}

template <typename T>
static int launch_abs_merge(const void* amax, const void* amin, int64_t in_ls, int d, int64_t n_seg,
                            const int32_t* sl, const int32_t* sb, const int32_t* se, int factor, int64_t m_in,
                            int64_t m_out, void* omax, void* omin, int64_t out_ls, cudaStream_t st) {
    const int64_t blocks = kvt::imax(1, kvt::imin((n_seg + 7) / 8, (int64_t)kvt::sm_count() * 16));
    abstract_merge_kernel<T><<<(unsigned)blocks, 256, 0, st>>>((const T*)amax, (const T*)amin, in_ls, d, n_seg, sl, sb,
                                                              se, factor, m_in, m_out, (T*)omax, (T*)omin, out_ls);
    return kvt_check_launch();
}

}  // namespace kvt

extern "C" int kvt_abstract_merge(const void* amax, const void* amin, int dtype, int64_t in_lane_stride, int d,
                                  int64_t n_seg, const int32_t* seg_lane, const int32_t* seg_begin,
                                  const int32_t* seg_end, int factor, int64_t m_in, int64_t m_out, void* amax_out,
                                  void* amin_out, int64_t out_lane_stride, void* stream) {
    if (!amax || !amin || !amax_out || !amin_out || d < 1 || n_seg < 0) return KVT_ERR_ARG;
    if (seg_lane ? (!seg_begin || !seg_end) : (factor < 1 || m_in < 0 || m_out < 1)) return KVT_ERR_ARG;
    if (n_seg == 0) return KVT_OK;
    cudaStream_t st = (cudaStream_t)stream;
#define KVT_M(T) return launch_abs_merge<T>(amax, amin, in_lane_stride, d, n_seg, seg_lane, seg_begin, seg_end, factor, \
                                             m_in, m_out, amax_out, amin_out, out_lane_stride, st)
    switch (dtype) {
        case KVT_F32: KVT_M(float);
        case KVT_F64: KVT_M(double);
        case KVT_BF16: KVT_M(__nv_bfloat16);
        case KVT_F16: KVT_M(__half);
        default: return KVT_ERR_DTYPE;
    }
#undef KVT_M
}
