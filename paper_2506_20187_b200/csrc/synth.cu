// Synthetic KV workload generator (bench / test input, not on the decode path).
//
// The planted-desert model of the reference generator (trace.py:270-315): per lane a unit
// direction u, a few hot token regions, key_t = a_t * u + noise_t and N(0,1)-like values,
// with desert amplitudes a_t ~ U(-0.25, 0.25) and hot amplitudes hot_base + U(0, 0.5).
// Unlike the reference (a sequential numpy PCG stream per lane, ~0.7 s per 64K lane on the
// host) every element here is a pure function of (lane seed, token, dim) through a counter
// hash, so a whole 64K x 256-lane layer is generated on the GPU in milliseconds AND any
// sampled lane can be regenerated bit-identically on the host (oracle/kvt_oracle.c
// ora_synth_lane) -- the bench's parity check and its CPU reference arm see exactly the
// tensors the GPU decoded.  Noise is not projected off u (its score contribution is
// ~0.05/sqrt(d) std, far below the desert/hot gap); normals are Irwin-Hall(4) of 16-bit
// uniforms, so the whole value recipe is exact integer math plus a fixed sequence of
// round-to-nearest f32 multiplies/adds (no contraction: __fmul_rn / __fadd_rn).
//
//   z(s, x)  = (sum of the four 16-bit halves of mix(s, 2x), mix(s, 2x+1)) * 2^-16 - 2   (exact)
//   n(s, x)  = z * f32(sqrt 3)                                                       (RN)
//   a_t      = r24(mix(s_a, t)) * span + base                                        (RN, RN)
//   key      = bf16_rn( (a_t * u_j) + (n(s_k, t*d+j) * noise_scale) )   planted
//            = bf16_rn( n(s_k, t*d+j) )                                  random
//   value    = bf16_rn( n(s_v, t*d+j) )
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace kvt {

__host__ __device__ __forceinline__ uint32_t synth_mix(uint32_t x) {  // lowbias32
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__host__ __device__ __forceinline__ uint32_t synth_hash(uint32_t s, uint32_t x) { return synth_mix(synth_mix(x) ^ s); }

__device__ __forceinline__ float synth_normal(uint32_t s, uint32_t x) {
    const uint32_t h0 = synth_hash(s, 2u * x), h1 = synth_hash(s, 2u * x + 1u);
    const uint32_t isum = (h0 & 0xffffu) + (h0 >> 16) + (h1 & 0xffffu) + (h1 >> 16);
    const float z = __fadd_rn(__fmul_rn((float)isum, 0x1p-16f), -2.0f);
    return __fmul_rn(z, 1.7320508075688772f);
}

// One thread = 8 consecutive dims of one token of one lane (one 16 B bf16 store per tensor).
__global__ void synth_layer_kernel(__nv_bfloat16* __restrict__ keys, __nv_bfloat16* __restrict__ values,
                                   int64_t lane_stride, int64_t n, int d, const uint32_t* __restrict__ lane_seed,
                                   const float* __restrict__ u, const int32_t* __restrict__ regions, int R,
                                   float desert_base, float desert_span, float hot_base, float hot_span,
                                   float noise_scale, int planted) {
    const int per_tok = d / 8;
    const int64_t lane = blockIdx.y;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n * per_tok) return;
    const int64_t t = gid / per_tok;
    const int j0 = (int)(gid % per_tok) * 8;
    const uint32_t ls = lane_seed[lane];
    const uint32_t s_k = synth_mix(ls ^ 0x9e3779b9u), s_v = synth_mix(ls ^ 0x85ebca6bu), s_a = synth_mix(ls ^ 0xc2b2ae35u);
    float a = 0.0f;
    if (planted) {
        bool hot = false;
        for (int r = 0; r < R; ++r) {
            const int32_t rs = regions[(lane * R + r) * 2], re = regions[(lane * R + r) * 2 + 1];
            hot |= (t >= rs && t < re);
        }
        const float r24 = __fmul_rn((float)(synth_hash(s_a, (uint32_t)t) >> 8), 0x1p-24f);
        a = hot ? __fadd_rn(__fmul_rn(r24, hot_span), hot_base) : __fadd_rn(__fmul_rn(r24, desert_span), desert_base);
    }
    __align__(16) __nv_bfloat16 kv[8], vv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int j = j0 + e;
        const uint32_t x = (uint32_t)(t * d + j);
        float k = synth_normal(s_k, x);
        if (planted) k = __fadd_rn(__fmul_rn(a, u[lane * d + j]), __fmul_rn(k, noise_scale));
        kv[e] = __float2bfloat16_rn(k);
        vv[e] = __float2bfloat16_rn(synth_normal(s_v, x));
    }
    const int64_t off = lane * lane_stride + t * d + j0;
    if (keys) *reinterpret_cast<uint4*>(keys + off) = *reinterpret_cast<const uint4*>(kv);
    if (values) *reinterpret_cast<uint4*>(values + off) = *reinterpret_cast<const uint4*>(vv);
}

}  // namespace kvt

extern "C" int kvt_synth_layer(void* keys, void* values, int64_t n_lanes, int64_t lane_stride, int64_t n, int d,
                               const uint32_t* lane_seed, const float* u, const int32_t* regions, int n_regions,
                               float desert_base, float desert_span, float hot_base, float hot_span,
                               float noise_scale, int planted, void* stream) {
    if ((!keys && !values) || !lane_seed || n_lanes < 0 || n < 0 || lane_stride < n * d) return KVT_ERR_ARG;
    if (planted && (!u || (n_regions > 0 && !regions) || n_regions < 0)) return KVT_ERR_ARG;
    if (d % 8 != 0 || d <= 0 || (uint64_t)n * (uint64_t)d >= (1ull << 31)) return KVT_ERR_SHAPE;
    if (n_lanes == 0 || n == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    if (((uintptr_t)keys | (uintptr_t)values | (uintptr_t)(lane_stride * 2)) % 16) return KVT_ERR_ARG;
    const int64_t threads = n * (d / 8);
    dim3 grid((unsigned)((threads + 255) / 256), (unsigned)n_lanes);
    kvt::synth_layer_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        (__nv_bfloat16*)keys, (__nv_bfloat16*)values, lane_stride, n, d, lane_seed, u, regions, n_regions,
        desert_base, desert_span, hot_base, hot_span, noise_scale, planted);
    return kvt_check_launch();
}
