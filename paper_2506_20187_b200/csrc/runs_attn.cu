// runs_attn.cu -- K6 runs scan / canonical partition and K7 sparse decode attention.
//
// K6: engine.py:176-183 _token_runs turns the (sorted) selected tokens into contiguous
// runs; the leaf shape that select_top_k + merge_desert leave behind (chunk_tree.py:
// 331-379) is those runs plus their complement (maximal desert runs).  One CTA per lane:
// flag run heads, block-scan run ids, emit (start, len) and the interleaved partition.
//
// K7: engine.py:145-154 attention_output = softmax(q.K_sel^T/sqrt d) @ V_sel.  The logits
// are the canonical f64 scores K5 already produced, so K is not re-read; only V rows of
// the selected tokens are gathered (ascending token order => runs are contiguous rows and
// each 128-dim bf16 row is one coalesced 256 B warp load).  Flash-decoding split: each CTA
// reduces a slice of the selected set to (m, l, o[d]) with f32 accumulation (f64 for f64
// values); the last split CTA of each lane (atomic ticket) rescales and combines the
// slices, so attention is one launch.  HBM-bound on k*d*s_V.
#include <type_traits>

#include <cstdlib>

#include "common.cuh"

namespace kvt {

constexpr int RUNS_THREADS = 512;

__global__ void __launch_bounds__(RUNS_THREADS) runs_kernel(
    const int32_t* __restrict__ sel_tok, const int32_t* __restrict__ n_sel, int64_t sel_stride, int64_t n,
    int32_t* __restrict__ run_start, int32_t* __restrict__ run_len, int64_t run_stride, int32_t* __restrict__ n_runs,
    int32_t* __restrict__ part_start, int8_t* __restrict__ part_state, int64_t part_stride,
    int32_t* __restrict__ n_part) {
    __shared__ long long scan_sh[33];
    const int tid = threadIdx.x;
    const int64_t li = blockIdx.x;
    const int64_t k = n_sel[li];
    const int32_t* tok = sel_tok + li * sel_stride;
    int32_t* rs = run_start + li * run_stride;
    int32_t* rl = run_len + li * run_stride;
    // pass 1: run heads -> run ids; store first position of each run in rl
    long long carry = 0;
    for (int64_t base = 0; base < k; base += RUNS_THREADS) {
        const int64_t i = base + tid;
        long long head = 0;
        if (i < k) head = (i == 0 || tok[i] != tok[i - 1] + 1) ? 1 : 0;
        long long tot;
        const long long ex = block_excl_scan<long long>(head, scan_sh, tot);
        if (head) {
            rs[carry + ex] = tok[i];
            rl[carry + ex] = (int32_t)i;
        }
        carry += tot;
    }
    const int64_t R = carry;
    __syncthreads();
    // pass 2: lengths from consecutive first positions (read r and r+1 before writing)
    for (int64_t base = 0; base < R; base += RUNS_THREADS) {
        const int64_t r = base + tid;
        int32_t f0 = 0, f1 = 0;
        if (r < R) { f0 = rl[r]; f1 = (r + 1 < R) ? rl[r + 1] : (int32_t)k; }
        __syncthreads();
        if (r < R) rl[r] = f1 - f0;
        __syncthreads();
    }
    if (tid == 0) n_runs[li] = (int32_t)R;
    if (!part_start) return;
    // pass 3: canonical partition = [gap0] run0 [gap1] run1 ... [gap_last]
    int32_t* ps = part_start + li * part_stride;
    int8_t* pst = part_state + li * part_stride;
    const long long pre = (R == 0) ? (n > 0 ? 1 : 0) : (rs[0] > 0 ? 1 : 0);
    if (tid == 0 && pre) { ps[0] = 0; pst[0] = 2; }
    long long carry2 = pre;
    for (int64_t base = 0; base < R; base += RUNS_THREADS) {
        const int64_t r = base + tid;
        long long cntl = 0;
        int32_t s = 0, e = 0, nxt = 0;
        if (r < R) {
            s = rs[r]; e = s + rl[r];
            nxt = (r + 1 < R) ? rs[r + 1] : (int32_t)n;
            cntl = 1 + (e < nxt ? 1 : 0);
        }
        long long tot;
        const long long ex = block_excl_scan<long long>(cntl, scan_sh, tot);
        if (r < R) {
            const int64_t p = carry2 + ex;
            ps[p] = s; pst[p] = 1;
            if (e < nxt) { ps[p + 1] = e; pst[p + 1] = 2; }
        }
        carry2 += tot;
    }
    if (tid == 0) n_part[li] = (int32_t)carry2;
}

// ------------------------------------------------------------------------------------------
// K7
// ------------------------------------------------------------------------------------------

constexpr int ATTN_THREADS = 256;
constexpr int ATTN_WARPS = ATTN_THREADS / 32;

template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

// softmax weight exp(x) of a (scaled, <= 0) logit difference, in the accumulation precision
template <typename Acc> __device__ __forceinline__ Acc softmax_w(double x);
template <> __device__ __forceinline__ float softmax_w<float>(double x) {
    return exp2f((float)(x * 1.4426950408889634));
}
template <> __device__ __forceinline__ double softmax_w<double>(double x) { return exp(x); }

template <typename T, bool VEC>
__device__ __forceinline__ void load_group_acc(const T* row, int g, int d, typename AccOf<T>::type v[4]) {
    const int j0 = 4 * g;
    if (VEC) {
        Elem<T>::load4f(row + j0, v);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = (j0 + i < d) ? Elem<T>::ld1f(row + j0 + i) : 0;
    }
}

// Last-arriving split CTA of a lane merges all splits' (m, l, o) (threadFenceReduction
// pattern: partial written -> __threadfence -> ticket; the last ticket holder reads all).
// The per-lane ticket counter is reset to 0 by the merger, so the workspace stays valid
// for the next call without a memset.
__device__ __forceinline__ void attn_finish(double* __restrict__ part, int splits, int d, int64_t li,
                                            unsigned int* __restrict__ tickets, float* __restrict__ out,
                                            double* __restrict__ out64, double scale) {
    __shared__ int s_last;
    __shared__ double s_scale[64];
    __shared__ double s_den, s_M;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(&tickets[li], 1u);
        s_last = (t == (unsigned)splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
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
        double* lse = part - 2 * (int64_t)gridDim.y;
        lse[2 * li] = s_M;
        lse[2 * li + 1] = den;
    }
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < splits; ++s) acc += s_scale[s] * __ldcg(P + s * (d + 2) + 2 + j);
        const double r = den > 0 ? acc / den : 0.0;
        if (out) out[li * d + j] = (float)r;
        if (out64) out64[li * d + j] = r;
    }
    if (threadIdx.x == 0) tickets[li] = 0;
}

// partial record per (lane, split): m (f64), l, o[d] (Acc); stored as doubles for simplicity
template <typename T, int G, bool VEC>
__global__ void __launch_bounds__(ATTN_THREADS) attn_split_kernel(
    const T* __restrict__ values, int64_t lane_stride, int d, const int32_t* __restrict__ sel_tok,
    const double* __restrict__ sel_score, const int32_t* __restrict__ n_sel, int64_t sel_stride, int splits,
    double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out,
    double* __restrict__ out64, double scale) {
    using Acc = typename AccOf<T>::type;
    __shared__ double red_m[ATTN_WARPS];
    __shared__ Acc red_o[ATTN_WARPS][4 * 32 * G];
    __shared__ Acc red_l[ATTN_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t li = blockIdx.y;
    const int s = blockIdx.x;
    const int64_t k = n_sel[li];
    const int64_t per = (k + splits - 1) / splits;
    const int64_t a = kvt::imin(k, s * per), b = kvt::imin(k, a + per);
    const int32_t* tok = sel_tok + li * sel_stride;
    const double* sc = sel_score + li * sel_stride;
    const T* base = values + li * lane_stride;
    // slice max
    double m = -INFINITY;
    for (int64_t i = a + threadIdx.x; i < b; i += ATTN_THREADS) m = fmax(m, sc[i]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(KVT_FULL, m, off));
    if (lane == 0) red_m[warp] = m;
    __syncthreads();
    m = red_m[0];
#pragma unroll
    for (int w = 1; w < ATTN_WARPS; ++w) m = fmax(m, red_m[w]);

    Acc o[G][4];
#pragma unroll
    for (int r = 0; r < G; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[r][i] = 0;
    Acc l = 0;
    constexpr int U = 4;
    int64_t i = a + warp;
    for (; i + (U - 1) * ATTN_WARPS < b; i += U * ATTN_WARPS) {
        Acc v[U][G][4];
        Acc w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ii = i + u * ATTN_WARPS;
            const T* row = base + (int64_t)tok[ii] * d;
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const int g = lane + 32 * r;
                if (4 * g < d) load_group_acc<T, VEC>(row, g, d, v[u][r]);
                else { v[u][r][0] = v[u][r][1] = v[u][r][2] = v[u][r][3] = 0; }
            }
            w[u] = softmax_w<Acc>((sc[ii] - m) * scale);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            l += w[u];
#pragma unroll
            for (int r = 0; r < G; ++r)
#pragma unroll
                for (int q = 0; q < 4; ++q) o[r][q] = fma(w[u], v[u][r][q], o[r][q]);
        }
    }
    for (; i < b; i += ATTN_WARPS) {
        const T* row = base + (int64_t)tok[i] * d;
        const Acc w = softmax_w<Acc>((sc[i] - m) * scale);
        l += w;
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const int g = lane + 32 * r;
            if (4 * g < d) {
                Acc v[4];
                load_group_acc<T, VEC>(row, g, d, v);
#pragma unroll
                for (int q = 0; q < 4; ++q) o[r][q] = fma(w, v[q], o[r][q]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < G; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) red_o[warp][4 * (lane + 32 * r) + q] = o[r][q];
    if (lane == 0) red_l[warp] = l;
    __syncthreads();
    double* P = part + ((int64_t)li * splits + s) * (d + 2);
    for (int j = threadIdx.x; j < d; j += ATTN_THREADS) {
        Acc acc = 0;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) acc += red_o[w][j];
        P[2 + j] = (double)acc;
    }
    if (threadIdx.x == 0) {
        Acc ls = 0;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) ls += red_l[w];
        P[0] = m;
        P[1] = (double)ls;
    }
    attn_finish(part, splits, d, li, tickets, out, out64, scale);
}

// Fast path: 16 B per lane per load, a row spans LPR = d*sizeof(T)/16 lanes, a warp
// instruction covers RPW = 32/LPR rows, and U = 8 instructions are in flight per lane
// (4 KB of V per warp for bf16 d=128).
template <typename T, int LPR>
__global__ void __launch_bounds__(ATTN_THREADS) attn_split16_kernel(
    const T* __restrict__ values, int64_t lane_stride, int d, const int32_t* __restrict__ sel_tok,
    const double* __restrict__ sel_score, const int32_t* __restrict__ n_sel, int64_t sel_stride, int splits,
    double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out,
    double* __restrict__ out64, double scale) {
    using Acc = typename AccOf<T>::type;
    constexpr int VPL = 16 / sizeof(T);
    constexpr int RPW = 32 / LPR;
    constexpr int U = 8;
    __shared__ double red_m[ATTN_WARPS];
    __shared__ Acc red_o[ATTN_WARPS][32 * VPL];
    __shared__ Acc red_l[ATTN_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / LPR, col = lane % LPR;
    const int64_t li = blockIdx.y;
    const int s = blockIdx.x;
    const int64_t k = n_sel[li];
    const int64_t per = (k + splits - 1) / splits;
    const int64_t a = kvt::imin(k, s * per), b = kvt::imin(k, a + per);
    const int32_t* tok = sel_tok + li * sel_stride;
    const double* sc = sel_score + li * sel_stride;
    const T* base = values + li * lane_stride + col * VPL;
    double m = -INFINITY;
    for (int64_t i = a + threadIdx.x; i < b; i += ATTN_THREADS) m = fmax(m, sc[i]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(KVT_FULL, m, off));
    if (lane == 0) red_m[warp] = m;
    __syncthreads();
    m = red_m[0];
#pragma unroll
    for (int w = 1; w < ATTN_WARPS; ++w) m = fmax(m, red_m[w]);

    Acc o[VPL];
#pragma unroll
    for (int e = 0; e < VPL; ++e) o[e] = 0;
    Acc l = 0;
    constexpr int STEP = ATTN_WARPS * RPW;  // rows per CTA instruction slot
    for (int64_t i0 = a + warp * RPW + sub; i0 < b; i0 += (int64_t)U * STEP) {
        uint4 raw[U];
        Acc w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + (int64_t)u * STEP;
            if (i < b) {
                raw[u] = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)tok[i] * d));
                w[u] = softmax_w<Acc>((sc[i] - m) * scale);
            } else {
                raw[u] = make_uint4(0, 0, 0, 0);
                w[u] = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            Acc v[VPL];
            const T* e = reinterpret_cast<const T*>(&raw[u]);
            if constexpr (sizeof(T) == 2) {
                float f[4];
                Elem<T>::unpack(make_uint2(raw[u].x, raw[u].y), f);
                v[0] = f[0]; v[1] = f[1]; v[2] = f[2]; v[3] = f[3];
                Elem<T>::unpack(make_uint2(raw[u].z, raw[u].w), f);
                v[4] = f[0]; v[5] = f[1]; v[6] = f[2]; v[7] = f[3];
            } else {
#pragma unroll
                for (int q = 0; q < VPL; ++q) v[q] = (Acc)e[q];
            }
            l += w[u];
#pragma unroll
            for (int q = 0; q < VPL; ++q) o[q] = fma(w[u], v[q], o[q]);
        }
    }
    // fold the RPW row groups of the warp onto lanes 0..LPR-1
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
        l += __shfl_xor_sync(KVT_FULL, l, off);
#pragma unroll
        for (int q = 0; q < VPL; ++q) o[q] += __shfl_xor_sync(KVT_FULL, o[q], off);
    }
    if (lane < LPR) {
#pragma unroll
        for (int q = 0; q < VPL; ++q) red_o[warp][lane * VPL + q] = o[q];
    }
    if (lane == 0) red_l[warp] = l;
    __syncthreads();
    double* P = part + ((int64_t)li * splits + s) * (d + 2);
    for (int j = threadIdx.x; j < d; j += ATTN_THREADS) {
        Acc acc = 0;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) acc += red_o[w][j];
        P[2 + j] = (double)acc;
    }
    if (threadIdx.x == 0) {
        Acc ls = 0;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) ls += red_l[w];
        P[0] = m;
        P[1] = (double)ls;
    }
    attn_finish(part, splits, d, li, tickets, out, out64, scale);
}

// INT4 values: a row (record) spans LPR = d/32 lanes, each lane dequantises one 32-dim
// group (16 B of codes + its (scale, min)) per row; RPW = 32/LPR rows per warp load.
template <int LPR>
__global__ void __launch_bounds__(ATTN_THREADS) attn_i4_kernel(
    const unsigned char* __restrict__ values, int64_t lane_stride_b, int d, const int32_t* __restrict__ sel_tok,
    const double* __restrict__ sel_score, const int32_t* __restrict__ n_sel, int64_t sel_stride, int splits,
    double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out,
    double* __restrict__ out64, double scale) {
    constexpr int RPW = 32 / LPR;
    constexpr int U = 4;
    __shared__ double red_m[ATTN_WARPS];
    __shared__ float red_o[ATTN_WARPS][32 * LPR];
    __shared__ float red_l[ATTN_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / LPR, grp = lane % LPR;
    const int rb = i4_row_bytes(d);
    const int64_t li = blockIdx.y;
    const int s = blockIdx.x;
    const int64_t k = n_sel[li];
    const int64_t per = (k + splits - 1) / splits;
    const int64_t a = kvt::imin(k, s * per), b = kvt::imin(k, a + per);
    const int32_t* tok = sel_tok + li * sel_stride;
    const double* sc = sel_score + li * sel_stride;
    const unsigned char* base = values + li * lane_stride_b;
    double m = -INFINITY;
    for (int64_t i = a + threadIdx.x; i < b; i += ATTN_THREADS) m = fmax(m, sc[i]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(KVT_FULL, m, off));
    if (lane == 0) red_m[warp] = m;
    __syncthreads();
    m = red_m[0];
#pragma unroll
    for (int w = 1; w < ATTN_WARPS; ++w) m = fmax(m, red_m[w]);

    float o[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) o[e] = 0.f;
    float l = 0.f, om = 0.f;
    constexpr int STEP = ATTN_WARPS * RPW;
    for (int64_t i0 = a + warp * RPW + sub; i0 < b; i0 += (int64_t)U * STEP) {
        uint4 cw[U];
        uint32_t pw[U];
        float w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + (int64_t)u * STEP;
            if (i < b) {
                const unsigned char* row = base + (int64_t)tok[i] * rb;
                cw[u] = __ldg(reinterpret_cast<const uint4*>(row + 16 * grp));
                pw[u] = __ldg(reinterpret_cast<const unsigned int*>(row + d / 2 + 4 * grp));
                w[u] = softmax_w<float>((sc[i] - m) * scale);
            } else {
                cw[u] = make_uint4(0, 0, 0, 0);
                pw[u] = 0;
                w[u] = 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // o += w * (c*scale + min) = (w*scale) * c + w*min: one FFMA per element, the
            // min term once per row (om); codes -> float by byte permute (0x4B0000cc = 2^23 + c)
            const __half2 p = *reinterpret_cast<const __half2*>(&pw[u]);
            const float ws = w[u] * __low2float(p);
            om = fmaf(w[u], __high2float(p), om);
            const uint32_t words[4] = {cw[u].x, cw[u].y, cw[u].z, cw[u].w};
            l += w[u];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t lo4 = words[q] & 0x0f0f0f0fu, hi4 = (words[q] >> 4) & 0x0f0f0f0fu;
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                    const float c0 = __uint_as_float(__byte_perm(0x4B000000u, lo4, 0x3004 + bb)) - 8388608.0f;
                    const float c1 = __uint_as_float(__byte_perm(0x4B000000u, hi4, 0x3004 + bb)) - 8388608.0f;
                    o[8 * q + 2 * bb] = fmaf(ws, c0, o[8 * q + 2 * bb]);
                    o[8 * q + 2 * bb + 1] = fmaf(ws, c1, o[8 * q + 2 * bb + 1]);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) o[e] += om;
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
        l += __shfl_xor_sync(KVT_FULL, l, off);
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] += __shfl_xor_sync(KVT_FULL, o[e], off);
    }
    if (lane < LPR) {
#pragma unroll
        for (int e = 0; e < 32; ++e) red_o[warp][32 * grp + e] = o[e];
    }
    if (lane == 0) red_l[warp] = l;
    __syncthreads();
    double* P = part + ((int64_t)li * splits + s) * (d + 2);
    for (int j = threadIdx.x; j < d; j += ATTN_THREADS) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) acc += red_o[w][j];
        P[2 + j] = (double)acc;
    }
    if (threadIdx.x == 0) {
        float ls = 0.f;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) ls += red_l[w];
        P[0] = m;
        P[1] = (double)ls;
    }
    attn_finish(part, splits, d, li, tickets, out, out64, scale);
}


// ---- gather attention v2 (the decode-path kernel for INT4 and 2-byte rows) ------------------
// Work unit = (lane, split) over <= R consecutive selected rows (R ~ 1024).  A row spans
// LPR lanes (one 16 B piece each); U row loads are in flight per lane.  Accumulation is
// packed f32x2 (sm_100a FFMA2/FADD2: two IEEE fmas per issue).
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// INT4 records: lane = one 32-dim group (16 B of codes + its (scale, min)).
// x^ = code * s + m, so sum_i w_i x^_ij = sum_i (w_i s_i) code_ij + sum_i w_i m_i: one packed
// fma per two codes; code -> float by byte permute into 2^23 + code and a packed subtract.
template <int D>
struct FmtI4 {
    static constexpr int LPR = D / 32, NE = 32;
    struct Raw { uint4 c; uint32_t sm; };
    __host__ __device__ static constexpr int row_bytes() { return D / 2 + D / 8; }
    __device__ static Raw load(const unsigned char* row, int grp) {
        Raw r;
        r.c = __ldg(reinterpret_cast<const uint4*>(row + 16 * grp));
        r.sm = __ldg(reinterpret_cast<const uint32_t*>(row + D / 2 + 4 * grp));
        return r;
    }
    __device__ static Raw zero() { Raw r; r.c = make_uint4(0, 0, 0, 0); r.sm = 0; return r; }
    // ring path: this lane's pieces of a row -> shared memory, and back
    __device__ static void issue(uint32_t srow, const unsigned char* grow, int grp) {
        cp_async16(srow + 16 * grp, grow + 16 * grp);
        cp_async4(srow + D / 2 + 4 * grp, grow + D / 2 + 4 * grp);
    }
    __device__ static Raw lds(const unsigned char* srow, int grp) {
        Raw r;
        r.c = *reinterpret_cast<const uint4*>(srow + 16 * grp);
        r.sm = *reinterpret_cast<const uint32_t*>(srow + D / 2 + 4 * grp);
        return r;
    }
    __device__ static void acc(uint64_t (&o2)[NE / 2], const Raw& r, float w, float& om) {
        const __half2 p = *reinterpret_cast<const __half2*>(&r.sm);
        const float ws = w * __low2float(p);
        om = fmaf(w, __high2float(p), om);
        const uint64_t ws2 = f2_pack(ws, ws), neg = f2_pack(-8388608.0f, -8388608.0f);
        const uint32_t words[4] = {r.c.x, r.c.y, r.c.z, r.c.w};
        // 2^23 + code as an f32 bit pattern: byte 3 = 0x4B from the magic word (first PRMT
        // source, a register), byte 0 = the code (second source); the selector stays an
        // immediate, so no per-use selector moves are issued
        const uint32_t magic = 0x4B000000u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t lo4 = words[q] & 0x0f0f0f0fu, hi4 = (words[q] >> 4) & 0x0f0f0f0fu;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const uint64_t c2 = f2_add(f2_pack(__uint_as_float(__byte_perm(magic, lo4, 0x3004 + bb)),
                                                   __uint_as_float(__byte_perm(magic, hi4, 0x3004 + bb))),
                                           neg);
                o2[4 * q + bb] = f2_fma(ws2, c2, o2[4 * q + bb]);
            }
        }
    }
    __device__ static float bias(float om) { return om; }
};

// 2-byte rows (bf16 / f16): lane = 8 consecutive dims (16 B).
template <typename T, int D>
struct Fmt16 {
    static constexpr int LPR = D * 2 / 16, NE = 8;
    using Raw = uint4;
    __host__ __device__ static constexpr int row_bytes() { return D * 2; }
    __device__ static Raw load(const unsigned char* row, int grp) {
        return __ldg(reinterpret_cast<const uint4*>(row + 16 * grp));
    }
    __device__ static Raw zero() { return make_uint4(0, 0, 0, 0); }
    __device__ static void issue(uint32_t srow, const unsigned char* grow, int grp) {
        cp_async16(srow + 16 * grp, grow + 16 * grp);
    }
    __device__ static Raw lds(const unsigned char* srow, int grp) {
        return *reinterpret_cast<const uint4*>(srow + 16 * grp);
    }
    __device__ static void acc(uint64_t (&o2)[NE / 2], const Raw& r, float w, float&) {
        const uint64_t w2 = f2_pack(w, w);
        const uint32_t words[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint64_t v2;
            if constexpr (std::is_same<T, __half>::value) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&words[i]));
                v2 = f2_pack(f.x, f.y);
            } else {
                v2 = f2_pack(__uint_as_float(words[i] << 16), __uint_as_float(words[i] & 0xffff0000u));
            }
            o2[i] = f2_fma(w2, v2, o2[i]);
        }
    }
    __device__ static float bias(float) { return 0.f; }
};

template <class F, int U>
__global__ void __launch_bounds__(ATTN_THREADS) attn_gather_kernel(
    const unsigned char* __restrict__ values, int64_t lane_stride_b, int d, const int32_t* __restrict__ sel_tok,
    const double* __restrict__ sel_score, const int32_t* __restrict__ n_sel, int64_t sel_stride, int splits, int R,
    double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out,
    double* __restrict__ out64, double scale, int kvg) {
    pdl_entry();
    // Each warp runs its own online softmax over rows warp*RPW + sub + u*STEP + it*U*STEP
    // (no block barrier before the first row load); the next iteration's token ids and
    // scores are fetched while the current rows are in flight.  Warps are combined in
    // shared memory at the end, then splits by the last-arriving CTA of the lane.
    constexpr int LPR = F::LPR, NE = F::NE, RPW = 32 / LPR, STEP = ATTN_WARPS * RPW;
    __shared__ double red_m[ATTN_WARPS];
    __shared__ float red_o[ATTN_WARPS][LPR * NE];
    __shared__ float red_l[ATTN_WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t li = blockIdx.y;
    const int s = blockIdx.x;
    const int64_t k = n_sel[li];
    const int64_t a = kvt::imin(k, (int64_t)s * R), b = kvt::imin(k, a + R);
    const int nr = (int)(b - a);
    const int32_t* tok = sel_tok + li * sel_stride + a;
    const double* sc = sel_score + li * sel_stride + a;
    const int sub = lane / LPR, grp = lane % LPR;
    const unsigned char* base = values + (li / kvg) * lane_stride_b;
    const double sl2 = scale * 1.4426950408889634;

    uint64_t o2[NE / 2];
#pragma unroll
    for (int e = 0; e < NE / 2; ++e) o2[e] = 0ull;
    float l = 0.f, om = 0.f;
    double m = -INFINITY;
    int t_nx[U];
    double s_nx[U];
    const int i0 = warp * RPW + sub;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = i0 + u * STEP;
        t_nx[u] = i < nr ? tok[i] : 0;
        s_nx[u] = i < nr ? sc[i] : -INFINITY;
    }
    for (int it = 0; it * U * STEP < nr; ++it) {  // warp-uniform trip count
        typename F::Raw raw[U];
        double sv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + (it * U + u) * STEP;
            raw[u] = i < nr ? F::load(base + (int64_t)t_nx[u] * F::row_bytes(), grp) : F::zero();
            sv[u] = s_nx[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {  // prefetch the next iteration's ids and scores
            const int i = i0 + ((it + 1) * U + u) * STEP;
            t_nx[u] = i < nr ? tok[i] : 0;
            s_nx[u] = i < nr ? sc[i] : -INFINITY;
        }
        double mi = sv[0];
#pragma unroll
        for (int u = 1; u < U; ++u) mi = fmax(mi, sv[u]);
#pragma unroll
        for (int off = 16; off >= LPR; off >>= 1) mi = fmax(mi, __shfl_xor_sync(KVT_FULL, mi, off));
        if (mi > m) {  // warp-uniform: rescale the running sums
            const float r = m == -INFINITY ? 0.f : exp2f((float)((m - mi) * sl2));
            const uint64_t r2 = f2_pack(r, r);
#pragma unroll
            for (int e = 0; e < NE / 2; ++e) o2[e] = f2_fma(o2[e], r2, 0ull);
            l *= r;
            om *= r;
            m = mi;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float w = sv[u] == -INFINITY ? 0.f : exp2f((float)((sv[u] - m) * sl2));
            F::acc(o2, raw[u], w, om);
            l += w;
        }
    }
    float o[NE];
#pragma unroll
    for (int e = 0; e < NE / 2; ++e) f2_unpack(o2[e], o[2 * e], o[2 * e + 1]);
    const float bias = F::bias(om);
#pragma unroll
    for (int e = 0; e < NE; ++e) o[e] += bias;
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
        l += __shfl_xor_sync(KVT_FULL, l, off);
#pragma unroll
        for (int e = 0; e < NE; ++e) o[e] += __shfl_xor_sync(KVT_FULL, o[e], off);
    }
    if (lane < LPR) {
#pragma unroll
        for (int e = 0; e < NE; ++e) red_o[warp][NE * grp + e] = o[e];
    }
    if (lane == 0) { red_l[warp] = l; red_m[warp] = m; }
    __syncthreads();
    double M = red_m[0];
#pragma unroll
    for (int w = 1; w < ATTN_WARPS; ++w) M = fmax(M, red_m[w]);
    float wsc[ATTN_WARPS];
#pragma unroll
    for (int w = 0; w < ATTN_WARPS; ++w) wsc[w] = red_m[w] == -INFINITY ? 0.f : exp2f((float)((red_m[w] - M) * sl2));
    double* P = part + ((int64_t)li * splits + s) * (d + 2);
    for (int j = tid; j < d; j += ATTN_THREADS) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) acc = fmaf(wsc[w], red_o[w][j], acc);
        P[2 + j] = (double)acc;
    }
    if (tid == 0) {
        float ls = 0.f;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) ls = fmaf(wsc[w], red_l[w], ls);
        P[0] = M;
        P[1] = (double)ls;
    }
    attn_finish(part, splits, d, li, tickets, out, out64, scale);
}

// Ring variant (the decode-path default): bytes in flight are not bounded by registers.
// Warp w owns a contiguous sub-range of the unit; it stages the sub-range's token ids and
// scores in shared memory (one coalesced pass, warp max taken there: no rescaling later),
// then streams its rows through a private S-slot ring with cp.async (each lane copies and
// later reads only its own 16 B pieces, so no intra-warp synchronisation is needed).
template <class F, int S>
__global__ void __launch_bounds__(ATTN_THREADS) attn_ring_kernel(
    const unsigned char* __restrict__ values, int64_t lane_stride_b, int d, const int32_t* __restrict__ sel_tok,
    const double* __restrict__ sel_score, const int32_t* __restrict__ n_sel, int64_t sel_stride, int splits, int R,
    double* __restrict__ part, unsigned int* __restrict__ tickets, float* __restrict__ out,
    double* __restrict__ out64, double scale, int kvg, const int32_t* __restrict__ ptable, int64_t ptable_stride,
    int pcrec) {
    pdl_entry();
    constexpr int LPR = F::LPR, NE = F::NE, RPW = 32 / LPR, RB = F::row_bytes(), SLOT = RPW * RB;
    extern __shared__ __align__(16) unsigned char ring_smem[];
    __shared__ double red_m[ATTN_WARPS];
    __shared__ float red_o[ATTN_WARPS][LPR * NE];
    __shared__ float red_l[ATTN_WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t li = blockIdx.y;
    const int s = blockIdx.x;
    const int64_t k = n_sel[li];
    const int64_t a = kvt::imin(k, (int64_t)s * R), b = kvt::imin(k, a + R);
    const int nr = (int)(b - a);
    const int per_w = (nr + ATTN_WARPS - 1) / ATTN_WARPS;
    const int wa = min(nr, warp * per_w), wb = min(nr, wa + per_w);
    unsigned char* ring = ring_smem + (size_t)warp * S * SLOT;
    int32_t* tok_s = reinterpret_cast<int32_t*>(ring_smem + (size_t)ATTN_WARPS * S * SLOT);
    float* w_s = reinterpret_cast<float*>(tok_s + R);
    const int32_t* tok = sel_tok + li * sel_stride + a;
    const double* sc = sel_score + li * sel_stride + a;
    double m = -INFINITY;
    // paged (hot tier): token -> pool row through the record table, resolved once here
    const int32_t* ptab = ptable ? ptable + (li / kvg) * ptable_stride : nullptr;
    for (int i = wa + lane; i < wb; i += 32) {
        int t = tok[i];
        if (ptab) {
            const int sl = ptab[t / pcrec];
            t = sl >= 0 ? sl * pcrec + t % pcrec : 0;
        }
        tok_s[i] = t;
        m = fmax(m, sc[i]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(KVT_FULL, m, off));
    const double sl2 = scale * 1.4426950408889634;
    __syncwarp();
    for (int i = wa + lane; i < wb; i += 32) w_s[i] = exp2f((float)((sc[i] - m) * sl2));  // once per row (L2 hit)
    __syncwarp();
    const int sub = lane / LPR, grp = lane % LPR;
    const unsigned char* base = ptable ? values : values + (li / kvg) * lane_stride_b;
    const uint32_t ring_a = (uint32_t)__cvta_generic_to_shared(ring);
    const int nslots = (wb - wa + RPW - 1) / RPW;
    uint64_t o2[NE / 2];
#pragma unroll
    for (int e = 0; e < NE / 2; ++e) o2[e] = 0ull;
    float l = 0.f, om = 0.f;
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {
        const int i = wa + j * RPW + sub;
        if (j < nslots && i < wb) F::issue(ring_a + j * SLOT + sub * RB, base + (int64_t)tok_s[i] * RB, grp);
        cp_async_commit();
    }
    for (int j = 0; j < nslots; ++j) {
        const int jn = j + S - 1;
        const int in = wa + jn * RPW + sub;
        if (jn < nslots && in < wb)
            F::issue(ring_a + (jn % S) * SLOT + sub * RB, base + (int64_t)tok_s[in] * RB, grp);
        cp_async_commit();
        cp_async_wait<S - 1>();
        const int i = wa + j * RPW + sub;
        if (i < wb) {
            const float w = w_s[i];
            F::acc(o2, F::lds(ring + (j % S) * SLOT + sub * RB, grp), w, om);
            l += w;
        }
    }
    cp_async_wait<0>();
    float o[NE];
#pragma unroll
    for (int e = 0; e < NE / 2; ++e) f2_unpack(o2[e], o[2 * e], o[2 * e + 1]);
    const float bias = F::bias(om);
#pragma unroll
    for (int e = 0; e < NE; ++e) o[e] += bias;
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
        l += __shfl_xor_sync(KVT_FULL, l, off);
#pragma unroll
        for (int e = 0; e < NE; ++e) o[e] += __shfl_xor_sync(KVT_FULL, o[e], off);
    }
    if (lane < LPR) {
#pragma unroll
        for (int e = 0; e < NE; ++e) red_o[warp][NE * grp + e] = o[e];
    }
    if (lane == 0) { red_l[warp] = l; red_m[warp] = m; }
    __syncthreads();
    double M = red_m[0];
#pragma unroll
    for (int w = 1; w < ATTN_WARPS; ++w) M = fmax(M, red_m[w]);
    float wsc[ATTN_WARPS];
#pragma unroll
    for (int w = 0; w < ATTN_WARPS; ++w) wsc[w] = red_m[w] == -INFINITY ? 0.f : exp2f((float)((red_m[w] - M) * sl2));
    double* P = part + ((int64_t)li * splits + s) * (d + 2);
    for (int j = tid; j < d; j += ATTN_THREADS) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) acc = fmaf(wsc[w], red_o[w][j], acc);
        P[2 + j] = (double)acc;
    }
    if (tid == 0) {
        float ls = 0.f;
#pragma unroll
        for (int w = 0; w < ATTN_WARPS; ++w) ls = fmaf(wsc[w], red_l[w], ls);
        P[0] = M;
        P[1] = (double)ls;
    }
    attn_finish(part, splits, d, li, tickets, out, out64, scale);
}

// Hot-tier paging context of kvt_sparse_decode_attn_paged (this host thread, one call).
struct PagedV {
    const int32_t* table = nullptr;
    int64_t stride = 0;
    int crec = 1;
};
static PagedV& paged_current() {
    static thread_local PagedV p;
    return p;
}

template <class F, int S>
static int launch_ring(const void* values, int64_t n_lanes, int64_t lane_stride_b, int d, const int32_t* sel_tok,
                       const double* sel_score, const int32_t* n_sel, int64_t sel_stride, int splits, int R,
                       double* part, unsigned int* tickets, float* out, double* out64, double scale,
                       cudaStream_t st) {
    constexpr int SLOT = (32 / F::LPR) * F::row_bytes();
    const size_t smem = (size_t)ATTN_WARPS * S * SLOT + (size_t)R * 8;
    KVT_PER_DEVICE(size_t, configured);
    if (smem > configured) {  // opt in for any size: static smem counts against the 48 KB default too
        cudaError_t e = cudaFuncSetAttribute(attn_ring_kernel<F, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        configured = smem;
    }
    dim3 grid(splits, (unsigned)n_lanes);
    const PagedV& pg = paged_current();
    launch_pdl(attn_ring_kernel<F, S>, grid, dim3(ATTN_THREADS), smem, st, (const unsigned char*)values, lane_stride_b, d, sel_tok,
                                                            sel_score, n_sel, sel_stride, splits, R, part, tickets,
                                                            out, out64, scale, kv_group_current(), pg.table, pg.stride,
                                                            pg.crec);
    return kvt_check_launch();
}

template <class F, int U>
static int launch_gather(const void* values, int64_t n_lanes, int64_t lane_stride_b, int d, const int32_t* sel_tok,
                         const double* sel_score, const int32_t* n_sel, int64_t sel_stride, int splits, int R,
                         double* part, unsigned int* tickets, float* out, double* out64, double scale,
                         cudaStream_t st) {
    dim3 grid(splits, (unsigned)n_lanes);
    launch_pdl(attn_gather_kernel<F, U>, grid, dim3(ATTN_THREADS), 0, st, (const unsigned char*)values, lane_stride_b, d, sel_tok,
                                                               sel_score, n_sel, sel_stride, splits, R, part, tickets,
                                                               out, out64, scale, kv_group_current());
    return kvt_check_launch();
}

}  // namespace kvt

using namespace kvt;

extern "C" int kvt_runs_scan(const int32_t* sel_tok, const int32_t* n_sel, int64_t sel_stride, int64_t n_lanes,
                             int64_t n, int32_t* run_start, int32_t* run_len, int64_t run_stride, int32_t* n_runs,
                             int32_t* part_start, int8_t* part_state, int64_t part_stride, int32_t* n_part,
                             void* stream) {
    if (!sel_tok || !n_sel || !run_start || !run_len || !n_runs || n_lanes < 0) return KVT_ERR_ARG;
    if (part_start && (!part_state || !n_part)) return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    runs_kernel<<<(unsigned)n_lanes, RUNS_THREADS, 0, (cudaStream_t)stream>>>(
        sel_tok, n_sel, sel_stride, n, run_start, run_len, run_stride, n_runs, part_start, part_state, part_stride,
        n_part);
    return kvt_check_launch();
}

// Workspace: one ticket counter per lane (first, 256 B aligned region), then the partials
// [n_lanes][splits][d + 2] f64.  The caller zero-fills it once; every call leaves the
// counters at zero again.
static inline size_t ticket_bytes(int64_t n_lanes) { return ((size_t)n_lanes * 4 + 255) & ~(size_t)255; }
extern "C" size_t kvt_attn_workspace_bytes(int64_t n_lanes, int d, int splits) {
    if (splits < 1) splits = 1;
    if (splits > 64) splits = 64;
    return ticket_bytes(n_lanes) + (size_t)n_lanes * 2 * sizeof(double) +
           (size_t)n_lanes * (size_t)splits * (size_t)(d + 2) * sizeof(double);
}

// After kvt_sparse_decode_attn, the workspace holds each lane's merged softmax state
// (m = max selected score, l = sum_i exp((s_i - m) logit_scale)): the partial a
// sequence shard contributes to the cross-rank log-sum-exp merge (kvt_lse_merge).
extern "C" int kvt_attn_lse(const void* ws, int64_t n_lanes, double* lse_out, void* stream) {
    if (!ws || !lse_out || n_lanes < 0) return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    const cudaError_t e = cudaMemcpyAsync(lse_out, (const char*)ws + ticket_bytes(n_lanes),
                                          (size_t)n_lanes * 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                                          (cudaStream_t)stream);
    return e == cudaSuccess ? KVT_OK : kvt_set_cuda_error(e);
}

// Cross-shard merge (config 5, after an all-gather): parts [P][n_lanes][d + 2] f64, each
// (m, l, o[d]) with o the shard's normalised output; out = sum_p w_p l_p o_p / sum_p w_p l_p,
// w_p = exp((m_p - max m) logit_scale); parts with l = 0 (no selected token) are skipped.
__global__ void lse_merge_kernel(const double* __restrict__ parts, int P, int64_t n_lanes, int d, double scale,
                                 float* __restrict__ out, double* __restrict__ out64) {
    const int64_t li = blockIdx.x;
    __shared__ double s_w[64];
    __shared__ double s_den;
    if (threadIdx.x < 32) {
        double M = -INFINITY;
        for (int p = threadIdx.x; p < P; p += 32) {
            const double* r = parts + ((int64_t)p * n_lanes + li) * (d + 2);
            if (r[1] > 0) M = fmax(M, r[0]);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) M = fmax(M, __shfl_xor_sync(KVT_FULL, M, off));
        double den = 0.0;
        for (int p = threadIdx.x; p < P; p += 32) {
            const double* r = parts + ((int64_t)p * n_lanes + li) * (d + 2);
            const double w = r[1] > 0 ? exp((r[0] - M) * scale) * r[1] : 0.0;
            s_w[p] = w;
            den += w;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) den += __shfl_xor_sync(KVT_FULL, den, off);
        if (threadIdx.x == 0) s_den = den;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double acc = 0.0;
        for (int p = 0; p < P; ++p) acc += s_w[p] * parts[((int64_t)p * n_lanes + li) * (d + 2) + 2 + j];
        const double r = s_den > 0 ? acc / s_den : 0.0;
        if (out) out[li * d + j] = (float)r;
        if (out64) out64[li * d + j] = r;
    }
}

extern "C" int kvt_lse_merge(const double* parts, int n_parts, int64_t n_lanes, int d, double logit_scale, float* out,
                             double* out64, void* stream) {
    if (!parts || (!out && !out64) || n_parts < 1 || n_parts > 64 || n_lanes < 0 || d < 1) return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    lse_merge_kernel<<<(unsigned)n_lanes, 128, 0, (cudaStream_t)stream>>>(parts, n_parts, n_lanes, d, logit_scale, out,
                                                                           out64);
    return kvt_check_launch();
}

static inline int agroups_for(int d) { return d <= 128 ? 1 : d <= 256 ? 2 : d <= 512 ? 4 : 0; }

template <typename T, int G, bool VEC>
static void launch_attn(const void* values, int64_t n_lanes, int64_t lane_stride, int d, const int32_t* sel_tok,
                        const double* sel_score, const int32_t* n_sel, int64_t sel_stride, int splits, double* part,
                        unsigned int* tickets, float* out, double* out64, double scale, cudaStream_t st) {
    dim3 grid(splits, (unsigned)n_lanes);
    attn_split_kernel<T, G, VEC><<<grid, ATTN_THREADS, 0, st>>>((const T*)values, lane_stride, d, sel_tok, sel_score,
                                                                n_sel, sel_stride, splits, part, tickets, out, out64, scale);
}

template <typename T>
static int dispatch_attn(const void* values, int64_t n_lanes, int64_t lane_stride, int d, const int32_t* sel_tok,
                         const double* sel_score, const int32_t* n_sel, int64_t sel_stride, int splits, double* part,
                         unsigned int* tickets, float* out, double* out64, double scale, cudaStream_t st) {
    const int64_t row = (int64_t)d * sizeof(T);
    const bool fast = ((uintptr_t)values % 16 == 0) && (lane_stride * (int64_t)sizeof(T)) % 16 == 0 &&
                      (row == 128 || row == 256 || row == 512);
    if (fast) {
        dim3 grid(splits, (unsigned)n_lanes);
        const int lpr = (int)(row / 16);
        if (lpr == 8)
            attn_split16_kernel<T, 8><<<grid, ATTN_THREADS, 0, st>>>((const T*)values, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride, splits, part, tickets, out, out64, scale);
        else if (lpr == 16)
            attn_split16_kernel<T, 16><<<grid, ATTN_THREADS, 0, st>>>((const T*)values, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride, splits, part, tickets, out, out64, scale);
        else
            attn_split16_kernel<T, 32><<<grid, ATTN_THREADS, 0, st>>>((const T*)values, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride, splits, part, tickets, out, out64, scale);
        return kvt_check_launch();
    }
    const bool vec = ((uintptr_t)values % (4 * sizeof(T)) == 0) && d % 4 == 0 && lane_stride % 4 == 0;
    switch (agroups_for(d)) {
#define KVT_CASE(GG)                                                                                                   \
    case GG:                                                                                                           \
        if (vec) launch_attn<T, GG, true>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride,     \
                                          splits, part, tickets, out, out64, scale, st);                               \
        else launch_attn<T, GG, false>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride, splits, \
                                       part, tickets, out, out64, scale, st);                                          \
        break;
        KVT_CASE(1) KVT_CASE(2) KVT_CASE(4)
#undef KVT_CASE
        default: return KVT_ERR_SHAPE;
    }
    return kvt_check_launch();
}

// Auto split count for the ring kernel: units of <= ATTN_RMAX rows.  A sweep over splits on the
// planted decode workload (tools/microbench.py attn; B200) shows per-unit fixed cost (staging,
// pipeline fill, partial merge) dominating any wave-tail effect: the fewest units that keep the
// staging bounded are best at k = 0.1 n and within ~8% at k = 0.5 n.
// INT4: 2400-row units through a 4-slot ring per warp (more resident CTAs beat deeper
// per-warp rings: config-3 A/B of slots x unit rows, tools/ab_libs.sh: 8 x 1664 2.69 ms,
// 6 x 1664 2.57, 4 x 1664 2.55, 3 x 1664 2.58, 2 x 1664 2.62, 4 x 1024 2.64, 4 x 2400 2.52).
// Few lanes (small batch): the fewest-units rule would leave most of the 148 SMs idle, so
// the split count is raised until the grid covers about two CTAs per SM, with units kept at
// >= 256 rows.
#ifndef KVT_ATTN_I4_S
#define KVT_ATTN_I4_S 4
#endif
#ifndef KVT_ATTN_I4_RMAX
#define KVT_ATTN_I4_RMAX 2400
#endif
static int ring_auto_splits(int64_t kmax, int v_dtype, int64_t n_lanes) {
    const int64_t rmax = v_dtype == KVT_I4 ? KVT_ATTN_I4_RMAX : 3328;
    const int64_t cap = kvt::imax(1, kvt::imin(64, (kmax + 31) / 32));
    int64_t s = kvt::imax(1, kvt::imin(cap, (kmax + rmax - 1) / rmax));
#ifndef KVT_ATTN_FILL
#define KVT_ATTN_FILL 2
#endif
    const int64_t fill = (KVT_ATTN_FILL * (int64_t)kvt::sm_count() + n_lanes - 1) / kvt::imax(1, n_lanes);
#ifndef KVT_ATTN_MINROWS
#define KVT_ATTN_MINROWS 256
#endif
    const int64_t by_rows = kvt::imax(1, kmax / KVT_ATTN_MINROWS);
    s = kvt::imax(s, kvt::imin(kvt::imin(fill, by_rows), cap));
    return (int)s;
}

extern "C" int kvt_sparse_decode_attn(const void* values, int v_dtype, int64_t n_lanes, int64_t lane_stride, int d,
                                      const int32_t* sel_tok, const double* sel_score, const int32_t* n_sel,
                                      int64_t sel_stride, double logit_scale, int splits, void* ws, float* out,
                                      double* out64, void* stream) {
    if (!values || !sel_tok || !sel_score || !n_sel || !ws || (!out && !out64) || d < 1 || n_lanes < 0)
        return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned int* tickets = (unsigned int*)ws;
    double* part = (double*)((char*)ws + ticket_bytes(n_lanes)) + 2 * n_lanes;  // after the lse slots
    int rc;
    const int64_t kmax = sel_stride;
    const int kvg = kv_group_current();
    if (splits <= 0) splits = ring_auto_splits(kmax, v_dtype, n_lanes);  // auto (the workspace must hold 64 splits)
    if (splits > 64) splits = 64;
    // rows per work unit: the whole selection in <= splits units
    const int R = (int)kvt::imax(32, ((kmax + splits - 1) / splits + 31) / 32 * 32);
    const bool aligned = ((uintptr_t)values % 16) == 0;
    switch (v_dtype) {
        case KVT_I4: {
            if ((d != 128 && d != 256) || !aligned || (lane_stride % 16)) return KVT_ERR_SHAPE;
            if (R <= 8192)  // cp.async ring (the unit's ids + weights staged: 8 B per row)
                rc = d == 128 ? launch_ring<FmtI4<128>, KVT_ATTN_I4_S>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel,
                                                           sel_stride, splits, R, part, tickets, out, out64, logit_scale, st)
                              : launch_ring<FmtI4<256>, 6>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel,
                                                           sel_stride, splits, R, part, tickets, out, out64, logit_scale, st);
            else
                rc = d == 128 ? launch_gather<FmtI4<128>, 4>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel,
                                                             sel_stride, splits, R, part, tickets, out, out64, logit_scale, st)
                              : launch_gather<FmtI4<256>, 2>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel,
                                                             sel_stride, splits, R, part, tickets, out, out64, logit_scale, st);
            break;
        }
        case KVT_BF16:
        case KVT_F16:
            if ((d == 128 || d == 256) && aligned && (lane_stride * 2) % 16 == 0) {
                const int64_t lsb = lane_stride * 2;
#define KVT_G(TT, DD) (R <= 8192 ? launch_ring<Fmt16<TT, DD>, 12>(values, n_lanes, lsb, d, sel_tok, sel_score, n_sel, \
                                                                  sel_stride, splits, R, part, tickets, out, out64, \
                                                                  logit_scale, st)                                      \
                                 : launch_gather<Fmt16<TT, DD>, 4>(values, n_lanes, lsb, d, sel_tok, sel_score, n_sel,  \
                                                                   sel_stride, splits, R, part, tickets, out, out64,    \
                                                                   logit_scale, st))
                if (v_dtype == KVT_BF16) rc = d == 128 ? KVT_G(__nv_bfloat16, 128) : KVT_G(__nv_bfloat16, 256);
                else rc = d == 128 ? KVT_G(__half, 128) : KVT_G(__half, 256);
#undef KVT_G
                break;
            }
            rc = v_dtype == KVT_BF16
                     ? dispatch_attn<__nv_bfloat16>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride,
                                                    splits, part, tickets, out, out64, logit_scale, st)
                     : dispatch_attn<__half>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride,
                                             splits, part, tickets, out, out64, logit_scale, st);
            break;
        case KVT_F32: rc = dispatch_attn<float>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride, splits, part, tickets, out, out64, logit_scale, st); break;
        case KVT_F64: rc = dispatch_attn<double>(values, n_lanes, lane_stride, d, sel_tok, sel_score, n_sel, sel_stride, splits, part, tickets, out, out64, logit_scale, st); break;
        default: return KVT_ERR_DTYPE;
    }
    return rc;
}

extern "C" int kvt_sparse_decode_attn_paged(const void* pool, const int32_t* table, int64_t table_stride, int crec,
                                            int64_t n_lanes, int d, const int32_t* sel_tok, const double* sel_score,
                                            const int32_t* n_sel, int64_t sel_stride, double logit_scale, int splits,
                                            void* ws, float* out, double* out64, void* stream) {
    if (!pool || !table || table_stride < 1 || crec < 1) return KVT_ERR_ARG;
    if ((d != 128 && d != 256) || ((uintptr_t)pool % 16)) return KVT_ERR_SHAPE;
    if (splits <= 0) splits = ring_auto_splits(sel_stride, KVT_I4, n_lanes);
    if (splits > 64) splits = 64;
    const int64_t R = kvt::imax(32, ((sel_stride + splits - 1) / splits + 31) / 32 * 32);
    if (R > 8192) return KVT_ERR_SHAPE;  // the ring path stages each unit's rows
    PagedV& pg = paged_current();
    pg.table = table;
    pg.stride = table_stride;
    pg.crec = crec;
    const int rc = kvt_sparse_decode_attn(pool, KVT_I4, n_lanes, 0, d, sel_tok, sel_score, n_sel, sel_stride,
                                          logit_scale, splits, ws, out, out64, stream);
    pg = PagedV();
    return rc;
}

// ---- live chunks of a selection (the skew behind adaptive chunk sizing) ----------------------
// Per lane and power-of-two chunk size 2^(lg0 + j), j < nlev: how many chunks of a uniform grid
// hold at least one selected token, counted from the lane's runs (ascending, disjoint): run r
// covers chunks [s >> lg, (e - 1) >> lg], minus one when it starts in the chunk where run r - 1
// ended.  The decoder turns these counts into the expected candidate tokens of each grid
// (chunk_tree.py:34-123 frames the same skew as the importance density rho).
__global__ void live_chunks_kernel(const int32_t* __restrict__ run_start, const int32_t* __restrict__ run_len,
                                   const int32_t* __restrict__ n_runs, int64_t run_stride, int lg0, int nlev,
                                   long long* __restrict__ out) {
    const int64_t li = blockIdx.x;
    const int nr = n_runs[li];
    const int32_t* rs = run_start + li * run_stride;
    const int32_t* rl = run_len + li * run_stride;
    long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
        const int s = rs[r], e = s + rl[r];
        const int pe = r > 0 ? rs[r - 1] + rl[r - 1] - 1 : -1;  // last token of the previous run
        for (int j = 0; j < nlev && j < 8; ++j) {
            const int lg = lg0 + j;
            const int a = s >> lg, b = (e - 1) >> lg;
            acc[j] += (long long)(b - a + 1) - (pe >= 0 && (pe >> lg) == a ? 1 : 0);
        }
    }
    __shared__ long long red[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < nlev && j < 8; ++j) {
        long long v = acc[j];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(KVT_FULL, v, o);
        if (lane == 0) red[j][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < nlev && threadIdx.x < 8) {
        long long v = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
        out[li * nlev + threadIdx.x] = v;
    }
}

extern "C" int kvt_live_chunks(const int32_t* run_start, const int32_t* run_len, const int32_t* n_runs,
                               int64_t run_stride, int64_t n_lanes, int lg0, int nlev, long long* out, void* stream) {
    if (!run_start || !run_len || !n_runs || !out || n_lanes < 0 || lg0 < 0 || nlev < 1 || nlev > 8 ||
        lg0 + nlev > 31)
        return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    live_chunks_kernel<<<(unsigned)n_lanes, 256, 0, (cudaStream_t)stream>>>(run_start, run_len, n_runs, run_stride,
                                                                          lg0, nlev, out);
    return kvt_check_launch();
}
