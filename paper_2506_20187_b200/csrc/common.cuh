// common.cuh -- shared device helpers for the kvtier B200 kernels (sm_100a).
//
// Canonical float64 dot product (the score definition shared with oracle/kvt_oracle.c,
// implemented independently there):
//   dim j is accumulated by warp lane (j >> 2) & 31 with an IEEE fma chain in increasing j,
//   then the 32 lane partials are combined by the fixed tree over lane bits 4,3,2,1,0
//   (xor-butterfly: pairs (l, l^16), then (l, l^8), ...).  fp32/bf16/fp16 inputs are exact
//   in f64, so products are exact and the result is bit-reproducible on the host.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kvtier_b200.h"

#define KVT_FULL 0xffffffffu

namespace kvt {

// Per-device host state.  Function attributes (the dynamic shared-memory opt-in), SM counts
// and occupancy are per device, and one process may drive several GPUs, so every one-time
// launch setup lives in a slot of the current device (cudaGetDevice).
constexpr int kMaxDevices = 64;
inline int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    return dev;
}
inline int sm_count() {
    static int sms[kMaxDevices] = {0};
    const int dev = current_device();
    if (sms[dev] <= 0) {
        if (cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms[dev] <= 0)
            sms[dev] = 148;
    }
    return sms[dev];
}
// `static T name = 0;` made per device: KVT_PER_DEVICE(bool, configured) binds `configured`
// to the current device's slot.
#define KVT_PER_DEVICE(T, name) \
    static T name##_slots_[::kvt::kMaxDevices] = {}; \
    T& name = name##_slots_[::kvt::current_device()]

template <typename A, typename B>
__host__ __device__ __forceinline__ int64_t imin(A a, B b) { return (int64_t)a < (int64_t)b ? (int64_t)a : (int64_t)b; }
template <typename A, typename B>
__host__ __device__ __forceinline__ int64_t imax(A a, B b) { return (int64_t)a > (int64_t)b ? (int64_t)a : (int64_t)b; }

// ------------------------------------------------------------------------------------------
// element loads (4 consecutive elements, widened)
// ------------------------------------------------------------------------------------------

template <typename T> struct Elem;
template <> struct Elem<float> {
    static constexpr int code = KVT_F32;
    __device__ __forceinline__ static void load4(const float* p, double v[4]) {
        float4 x = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    __device__ __forceinline__ static void load4f(const float* p, float v[4]) {
        float4 x = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    __device__ __forceinline__ static double ld1(const float* p) { return (double)__ldg(p); }
    __device__ __forceinline__ static float ld1f(const float* p) { return __ldg(p); }
};
template <> struct Elem<double> {
    static constexpr int code = KVT_F64;
    __device__ __forceinline__ static void load4(const double* p, double v[4]) {
        double2 a = __ldg(reinterpret_cast<const double2*>(p));
        double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    __device__ __forceinline__ static void load4f(const double* p, double v[4]) { load4(p, v); }
    __device__ __forceinline__ static double ld1(const double* p) { return __ldg(p); }
    __device__ __forceinline__ static double ld1f(const double* p) { return __ldg(p); }
};
template <> struct Elem<__nv_bfloat16> {
    static constexpr int code = KVT_BF16;
    __device__ __forceinline__ static void unpack(uint2 u, float f[4]) {
        f[0] = __uint_as_float(u.x << 16);
        f[1] = __uint_as_float(u.x & 0xffff0000u);
        f[2] = __uint_as_float(u.y << 16);
        f[3] = __uint_as_float(u.y & 0xffff0000u);
    }
    __device__ __forceinline__ static void load4(const __nv_bfloat16* p, double v[4]) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        float f[4];
        unpack(u, f);
        v[0] = f[0]; v[1] = f[1]; v[2] = f[2]; v[3] = f[3];
    }
    __device__ __forceinline__ static void load4f(const __nv_bfloat16* p, float v[4]) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        unpack(u, v);
    }
    __device__ __forceinline__ static double ld1(const __nv_bfloat16* p) { return (double)__bfloat162float(p[0]); }
    __device__ __forceinline__ static float ld1f(const __nv_bfloat16* p) { return __bfloat162float(p[0]); }
};
template <> struct Elem<__half> {
    static constexpr int code = KVT_F16;
    __device__ __forceinline__ static void unpack(uint2 u, float f[4]) {
        __half2 a = *reinterpret_cast<__half2*>(&u.x), b = *reinterpret_cast<__half2*>(&u.y);
        float2 fa = __half22float2(a), fb = __half22float2(b);
        f[0] = fa.x; f[1] = fa.y; f[2] = fb.x; f[3] = fb.y;
    }
    __device__ __forceinline__ static void load4(const __half* p, double v[4]) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        __half2 a = *reinterpret_cast<__half2*>(&u.x), b = *reinterpret_cast<__half2*>(&u.y);
        float2 fa = __half22float2(a), fb = __half22float2(b);
        v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
    }
    __device__ __forceinline__ static void load4f(const __half* p, float v[4]) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        __half2 a = *reinterpret_cast<__half2*>(&u.x), b = *reinterpret_cast<__half2*>(&u.y);
        float2 fa = __half22float2(a), fb = __half22float2(b);
        v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
    }
    __device__ __forceinline__ static double ld1(const __half* p) { return (double)__half2float(p[0]); }
    __device__ __forceinline__ static float ld1f(const __half* p) { return __half2float(p[0]); }
};

// Load the (up to) 4 dims of group g of row `row` (d dims).  VEC: d % 4 == 0 and aligned.
template <typename T, bool VEC>
__device__ __forceinline__ void load_group(const T* row, int g, int d, double v[4]) {
    int j0 = 4 * g;
    if (VEC) {
        Elem<T>::load4(row + j0, v);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = (j0 + i < d) ? Elem<T>::ld1(row + j0 + i) : 0.0;
    }
}

// Same, from shared memory (plain vector loads).
template <typename T> __device__ __forceinline__ void lds4(const T* p, double v[4]);
template <> __device__ __forceinline__ void lds4<float>(const float* p, double v[4]) {
    float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
template <> __device__ __forceinline__ void lds4<double>(const double* p, double v[4]) {
    double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
template <> __device__ __forceinline__ void lds4<__nv_bfloat16>(const __nv_bfloat16* p, double v[4]) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    float f[4];
    Elem<__nv_bfloat16>::unpack(u, f);
    v[0] = f[0]; v[1] = f[1]; v[2] = f[2]; v[3] = f[3];
}
template <> __device__ __forceinline__ void lds4<__half>(const __half* p, double v[4]) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    __half2 a = *reinterpret_cast<__half2*>(&u.x), b = *reinterpret_cast<__half2*>(&u.y);
    float2 fa = __half22float2(a), fb = __half22float2(b);
    v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
}

// ------------------------------------------------------------------------------------------
// INT4 KV records (kvt_kv_quant): per token d/2 code bytes (dim 2j low nibble, 2j+1 high
// nibble) followed by d/32 (scale, min) fp16 pairs; x^ = fmaf(code, scale, min).
// ------------------------------------------------------------------------------------------

struct I4 {};  // storage tag

__host__ __device__ __forceinline__ int i4_row_bytes(int d) { return d / 2 + (d / 32) * 4; }

__device__ __forceinline__ void i4_dequant4(uint32_t c16, __half2 p, float f[4]) {
    const float s = __low2float(p), m = __high2float(p);
    f[0] = __fmaf_rn((float)(c16 & 15u), s, m);
    f[1] = __fmaf_rn((float)((c16 >> 4) & 15u), s, m);
    f[2] = __fmaf_rn((float)((c16 >> 8) & 15u), s, m);
    f[3] = __fmaf_rn((float)((c16 >> 12) & 15u), s, m);
}

// Row loaders on byte-addressed rows (shared or global memory): dims 4g..4g+3 as f64.
template <typename T> struct RowLd {
    __host__ __device__ static int row_bytes(int d) { return d * (int)sizeof(T); }
    __device__ __forceinline__ static void load(const unsigned char* row, int g, int d, double v[4]) {
        lds4<T>(reinterpret_cast<const T*>(row) + 4 * g, v);
    }
    __device__ __forceinline__ static void loadf(const unsigned char* row, int g, int d, float v[4]) {
        const T* p = reinterpret_cast<const T*>(row) + 4 * g;
        if constexpr (sizeof(T) == 4) {
            const float4 x = *reinterpret_cast<const float4*>(p);
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
            Elem<T>::unpack(*reinterpret_cast<const uint2*>(p), v);
        }
    }
};
template <> struct RowLd<I4> {
    __host__ __device__ static int row_bytes(int d) { return i4_row_bytes(d); }
    __device__ __forceinline__ static void load(const unsigned char* row, int g, int d, double v[4]) {
        const uint32_t c = *reinterpret_cast<const unsigned short*>(row + 2 * g);
        const __half2 p = *reinterpret_cast<const __half2*>(row + d / 2 + 4 * (g >> 3));
        float f[4];
        i4_dequant4(c, p, f);
        v[0] = f[0]; v[1] = f[1]; v[2] = f[2]; v[3] = f[3];
    }
    __device__ __forceinline__ static void loadf(const unsigned char* row, int g, int d, float v[4]) {
        const uint32_t c = *reinterpret_cast<const unsigned short*>(row + 2 * g);
        const __half2 p = *reinterpret_cast<const __half2*>(row + d / 2 + 4 * (g >> 3));
        i4_dequant4(c, p, v);
    }
};

// Orderable 32-bit key of a finite float (larger value -> larger key); -0 == +0.
__device__ __forceinline__ uint32_t ord_key32(float s) {
    if (s == 0.0f) s = 0.0f;
    const uint32_t b = __float_as_uint(s);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key32_to_float(uint32_t k) {
    const uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(b);
}

// ------------------------------------------------------------------------------------------
// canonical reductions
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ double tree_allreduce(double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(KVT_FULL, v, off);
    return v;
}

// Reduce-scatter of 8 per-lane partials (tokens 0..7) with the canonical tree; on return
// lane L holds the full dot of token (L >> 2) & 7 (same value on the 4 lanes of a quad).
template <typename V>
__device__ __forceinline__ V tree_8tok(V p[8], int lane) {
    {
        const bool b = lane & 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            V send = b ? p[i] : p[4 + i];
            V keep = b ? p[4 + i] : p[i];
            p[i] = keep + __shfl_xor_sync(KVT_FULL, send, 16);
        }
    }
    {
        const bool b = lane & 8;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            V send = b ? p[i] : p[2 + i];
            V keep = b ? p[2 + i] : p[i];
            p[i] = keep + __shfl_xor_sync(KVT_FULL, send, 8);
        }
    }
    {
        const bool b = lane & 4;
        V send = b ? p[0] : p[1];
        V keep = b ? p[1] : p[0];
        p[0] = keep + __shfl_xor_sync(KVT_FULL, send, 4);
    }
    V v = p[0];
    v = v + __shfl_xor_sync(KVT_FULL, v, 2);
    v = v + __shfl_xor_sync(KVT_FULL, v, 1);
    return v;
}

// Same for 4 partials: lane L ends with the full dot of item (L >> 3) & 3.
__device__ __forceinline__ double tree_4tok(double p[4], int lane) {
    {
        const bool b = lane & 16;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            double send = b ? p[i] : p[2 + i];
            double keep = b ? p[2 + i] : p[i];
            p[i] = keep + __shfl_xor_sync(KVT_FULL, send, 16);
        }
    }
    {
        const bool b = lane & 8;
        double send = b ? p[0] : p[1];
        double keep = b ? p[1] : p[0];
        p[0] = keep + __shfl_xor_sync(KVT_FULL, send, 8);
    }
    double v = p[0];
    v = v + __shfl_xor_sync(KVT_FULL, v, 4);
    v = v + __shfl_xor_sync(KVT_FULL, v, 2);
    v = v + __shfl_xor_sync(KVT_FULL, v, 1);
    return v;
}

// Chain length (<= 4*ceil(d/128)) + tree depth; the soundness widening factor.
__host__ __device__ __forceinline__ int chain_len(int d) { return 4 * ((d + 127) / 128) + 5; }
__host__ __device__ __forceinline__ double slack_factor(int d) {
    return (double)(2 * chain_len(d) + 4) * 0x1p-53;
}

// Orderable 64-bit key of a finite double (larger score -> larger key); -0 == +0.
__device__ __forceinline__ uint64_t ord_key(double s) {
    if (s == 0.0) s = 0.0;
    uint64_t b = (uint64_t)__double_as_longlong(s);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_to_double(uint64_t k) {
    uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// ------------------------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, cp.async.bulk) helpers
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (16 B aligned, bytes % 16 == 0), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------------------------------------
// block-level scans (blockDim.x multiple of 32, <= 1024)
// ------------------------------------------------------------------------------------------

template <typename V>
__device__ __forceinline__ V warp_incl_scan(V v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        V t = __shfl_up_sync(KVT_FULL, v, off);
        if (lane >= off) v += t;
    }
    return v;
}

// Exclusive scan across the block; returns this thread's exclusive prefix and the total.
// `sh` must hold >= 33 V.  Contains __syncthreads().
template <typename V>
__device__ __forceinline__ V block_excl_scan(V v, V* sh, V& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    V inc = warp_incl_scan(v, lane);
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        V w = lane < nw ? sh[lane] : V(0);
        V wi = warp_incl_scan(w, lane);
        if (lane < nw) sh[lane] = wi - w;
        if (lane == 31) sh[32] = wi;
    }
    __syncthreads();
    V res = sh[warp] + inc - v;
    total = sh[32];
    __syncthreads();
    return res;
}

}  // namespace kvt

bool kvt_fast_ok(int key_dtype, int d);

// INT4 K1 (quant.cu)
int kvt_abstract_build_i4(const void* keys, int64_t n_lanes, int64_t lane_stride_b, int64_t n, int d, int C,
                          int64_t c_begin, int64_t c_end, void* amax, void* amin, int64_t abs_lane_stride, bool bf,
                          cudaStream_t st);

// GQA: query lane i reads the K/V/abstracts of lane i / kv_group (LLaMA-3 layout: the query
// heads of one KV head are adjacent).  kvt_select_attend sets the group for the launches it
// makes through this host thread-local scope; the standalone entry points run with 1.
int& kv_group_tls();
struct KvGroupScope {
    int saved;
    explicit KvGroupScope(int g) : saved(kv_group_tls()) { kv_group_tls() = g > 1 ? g : 1; }
    ~KvGroupScope() { kv_group_tls() = saved; }
};
inline int kv_group_current() { return kv_group_tls(); }
// GQA union candidates (kvt_select_attend, INT4 keys): the plan emits one candidate list per
// KV lane (the union over its query lanes) and the scorer writes the candidates' token ids
// once per group, in the row of the group's first query lane; the selectors read row
// (i / g) * g.  1 = one list per query lane.
int& cand_group_tls();
// Per-lane selection hints (the previous step's k-th estimate, kvt_layer_args.sel_hint) for the
// K5 launches of kvt_select_attend on this host thread; nullptr = none.
float*& sel_hint_tls();
struct SelHintScope {
    float* saved;
    explicit SelHintScope(float* h) : saved(sel_hint_tls()) { sel_hint_tls() = h; }
    ~SelHintScope() { sel_hint_tls() = saved; }
};
inline float* sel_hint_current() { return sel_hint_tls(); }
struct CandGroupScope {
    int saved;
    explicit CandGroupScope(int g) : saved(cand_group_tls()) { cand_group_tls() = g > 1 ? g : 1; }
    ~CandGroupScope() { cand_group_tls() = saved; }
};
inline int cand_group_current() { return cand_group_tls(); }

// Programmatic dependent launch (decode-path kernels): a kernel launched with
// launch_pdl may start while its predecessor drains; pdl_entry() -- the first statement of
// every such kernel -- waits for the predecessor grid (and its memory) before anything is
// read, then lets the successor launch.  Launch latency overlaps the predecessor's tail.
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Resident CTAs per SM of `kernel` at this block size / dynamic smem (occupancy API), so
// persistent grids are exactly one wave.  Falls back to `fallback` on error.
template <typename K>
inline int resident_per_sm(K kernel, int threads, size_t smem, int fallback) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return fallback;
    }
    return n;
}

// GQA union attention over INT4 values (attn_gqa.cu); KVT_ERR_ARG = shape not covered
extern "C" int kvt_sparse_decode_attn_gqa(const void* values, int64_t n_lanes, int64_t lane_stride_b, int d, int kvg,
                                          int64_t n_ctx, const int32_t* sel_tok, const double* sel_score,
                                          const int32_t* n_sel, int64_t sel_stride, double logit_scale, void* ws,
                                          void* scratch, size_t scratch_bytes, float* out, double* out64,
                                          void* stream);
extern "C" size_t kvt_attn_gqa_scratch_bytes(int64_t n_lanes, int kvg, int64_t n_ctx);

// status plumbing (api.cu)
int kvt_set_error_text(const char* msg);
int kvt_set_cuda_error(cudaError_t e);
int kvt_check_launch();
