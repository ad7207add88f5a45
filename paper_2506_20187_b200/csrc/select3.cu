// select3.cu -- K5 (fast path): exact canonical top-k from K4's f32 estimates, one CTA per lane.
//
// The plan supplies, per lane, E (a rigorous bound on |f32 estimate s - canonical f64 dot c|
// for every candidate), tau (<= the k-th canonical dot) and Umax (>= every candidate's c).
// 1. Histogram the estimates into 4096 linear buckets over [tau - 2E, Umax + 2E] (the range
//    adapts to the lane's score spread); the bucket holding the k-th estimate is found by a
//    block scan, its members gathered into shared memory and radix-selected (32-bit keys) to
//    get the exact k-th largest estimate T.
// 2. s > T + 2E  =>  c > S_k (selected);  s < T - 2E  =>  c < S_k (not selected): only the
//    band [T - 2E, T + 2E] -- typically a handful of tokens -- is re-scored canonically in
//    f64 from the key rows and ranked by (c desc, token asc) to fill the remaining slots.
// 3. Stable warp-ballot compaction writes the set in ascending token order; the run scan
//    (engine.py:176-183) is fused.
// A wide band or an overfull bucket (heavy ties) takes the exact fallback: canonical f64
// re-scoring of every candidate into `scratch` and a 64-bit radix select over it.  The
// result is always the oracle's canonical top-k set (score desc, index asc).
#include <type_traits>

#include "common.cuh"

namespace kvt {

constexpr int S3_THREADS_MAX = 1024;  // CTA size: 512 (two CTAs per SM: a 256-lane layer is one
// wave) or 1024 when the layer has fewer lanes than SMs (each lane's passes split over 32 warps)
constexpr int S3_WARPS_MAX = S3_THREADS_MAX / 32;
constexpr int S3_BINS = 4096;
constexpr int S3_LIST_CAP = 8192;
constexpr int S3_BAND_CAP = 1024;
constexpr int S3_UB = 8;  // float4 loads in flight per thread (block-strided passes)
constexpr int S3_UW = 4;
#ifndef KVT_S3_UWC
#define KVT_S3_UWC 2
#endif
constexpr int S3_UWC = KVT_S3_UWC;  // windows per warp iteration of the compaction pass: its
// per-window work (scan, carries, stores) is the critical path, so fewer windows in flight (fewer
// live registers) is faster -- layer-2 compaction 19.3 us at 4, 15.5-15.7 us at 1-2, 34.6 at 8

// Phase timestamps (development aid, off unless kvt_debug_select_phases set a buffer):
// thread 0 of CTA b writes %globaltimer at phase p to buf[b * 8 + p].
__device__ unsigned long long* g_s3_phase = nullptr;
__device__ __forceinline__ void s3_mark(int p) {
    unsigned long long* P = g_s3_phase;
    if (P && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P[blockIdx.x * 8 + p] = t;
    }
}

struct S3Shared {
    unsigned int hist[S3_BINS];
    double band_c[S3_BAND_CAP];
    int band_t[S3_BAND_CAP];
    unsigned char band_sel[S3_BAND_CAP];
    unsigned int rh[256];
    long long scan_sh[33];
    long long warp_cnt[S3_WARPS_MAX];
    unsigned long long prefix, mask;
    unsigned int list_n, remaining;
    int bstar;
    long long above;
};

// Bucket of an estimate: any deterministic non-decreasing map works (the exact k-th value
// comes from the bucket's own list), so f32 arithmetic is enough.
__device__ __forceinline__ int s3_bucket(float s, float lo, float inv) {
    if (!(s >= lo)) return -1;
    const float x = (s - lo) * inv;
    return x >= (float)(S3_BINS - 1) ? S3_BINS - 1 : (int)x;
}

// Block-wide: find the digit bin of `hist` (nb bins, descending order) where the running
// count from the top reaches `want`; returns (bin, count strictly above it) via S.
template <int NT>
__device__ __forceinline__ void s3_find_bin(S3Shared& S, const unsigned int* hist, int nb, long long want) {
    const int tid = threadIdx.x;
    const int per = (nb + NT - 1) / NT;
    long long loc = 0;
    for (int j = 0; j < per; ++j) {
        const int b = nb - 1 - (tid * per + j);
        if (b >= 0) loc += hist[b];
    }
    long long tot;
    const long long ex = block_excl_scan<long long>(loc, S.scan_sh, tot);
    if (ex < want && want <= ex + loc) {
        long long run = ex;
        for (int j = 0; j < per; ++j) {
            const int b = nb - 1 - (tid * per + j);
            if (b < 0) break;
            if (run + hist[b] >= want) {
                S.bstar = b;
                S.above = run;
                break;
            }
            run += hist[b];
        }
    }
    __syncthreads();
}

// Radix select on the shared list of 32-bit keys: exact key of the `want`-th largest.
// Short lists (the usual case: one of 4096 buckets) are ranked by counting instead: one
// barrier instead of four radix rounds.
template <int NT>
__device__ __forceinline__ uint32_t s3_list_select(S3Shared& S, const uint32_t* keys, int n, long long want) {
    const int tid = threadIdx.x, lane = tid & 31;
    if (n <= 128) {
        for (int j = tid; j < n; j += NT) {
            const uint32_t kj = keys[j];
            int gt = 0, eq = 0;
            for (int f = 0; f < n; ++f) {
                const uint32_t kf = keys[f];
                gt += kf > kj;
                eq += kf == kj;
            }
            if (gt < want && want <= gt + eq) S.prefix = kj;  // every writer stores the same key
        }
        __syncthreads();
        return (uint32_t)S.prefix;
    }
    if (tid == 0) { S.prefix = 0; S.mask = 0; S.remaining = (unsigned)want; }
    __syncthreads();
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += NT) S.rh[i] = 0;
        __syncthreads();
        const uint32_t pf = (uint32_t)S.prefix, mk = (uint32_t)S.mask;
        for (int base = 0; base < n; base += NT) {
            const int i = base + tid;
            int dg = 256;
            if (i < n && (keys[i] & mk) == pf) dg = (keys[i] >> shift) & 0xff;
            const unsigned peers = __match_any_sync(KVT_FULL, dg);
            if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&S.rh[dg], (unsigned)__popc(peers));
        }
        __syncthreads();
        if (tid < 32) {
            unsigned loc[8], ls = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) { loc[i] = S.rh[255 - 8 * lane - i]; ls += loc[i]; }
            const unsigned inc = warp_incl_scan(ls, lane), exc = inc - ls, rem = S.remaining;
            __syncwarp();  // every lane has read S.remaining before it is rewritten
            if (exc < rem && rem <= inc) {
                unsigned run = exc;
                for (int i = 0; i < 8; ++i) {
                    if (run + loc[i] >= rem) {
                        const int b = 255 - 8 * lane - i;
                        S.prefix = pf | ((uint32_t)b << shift);
                        S.mask = mk | (0xffu << shift);
                        S.remaining = rem - run;
                        break;
                    }
                    run += loc[i];
                }
            }
        }
        __syncthreads();
    }
    return (uint32_t)S.prefix;
}

// Stable warp-ballot compaction helper: warp w owns the contiguous range
// [w*per, (w+1)*per) of [0, n) and walks it 32 elements at a time.
template <int NW>
struct WarpRange {
    int64_t a, b;
    __device__ WarpRange(int64_t n, int warp) {
        const int64_t per = ((n + NW - 1) / NW + 31) / 32 * 32;
        a = kvt::imin(n, warp * per);
        b = kvt::imin(n, a + per);
    }
};

template <typename QT, typename T>
__device__ __forceinline__ double s3_canon(const QT* q, const unsigned char* row, int d, int lane) {
    double acc = 0.0;
    for (int g = lane; 4 * g < d; g += 32) {
        double v[4];
        RowLd<T>::load(row, g, d, v);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (4 * g + e < d) acc = fma((double)q[4 * g + e], v[e], acc);
    }
    return tree_allreduce(acc);
}

// Per-warp contiguous ranges in units of 128 elements (32 lanes x float4), so a warp's
// iteration covers 128 consecutive candidates and lane l owns elements 4l..4l+3 of it.
template <int NW>
struct WarpRange4 {
    int a, b;  // candidate counts are < 2^31: 32-bit indices in the hot loops
    __device__ WarpRange4(int64_t n, int warp) {
        const int per = (int)(((n + NW - 1) / NW + 127) / 128 * 128);
        a = (int)kvt::imin(n, (int64_t)warp * per);
        b = (int)kvt::imin(n, (int64_t)a + per);
    }
};

__device__ __forceinline__ void load4s(const float* sc, int i, int end, bool vec, float v[4]) {
    if (vec && i + 4 <= end) {
        const float4 x = *reinterpret_cast<const float4*>(sc + i);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (i + e < end) ? sc[i + e] : -INFINITY;
    }
}

template <typename QT, typename T, int NT>
__global__ void __launch_bounds__(NT, NT == 512 ? 2 : 1) topk_select3_kernel(
    const float* __restrict__ cs32, const int32_t* __restrict__ ctok, const int32_t* __restrict__ n_cand,
    int64_t cand_stride, const double* __restrict__ rec, int64_t k, const QT* __restrict__ q,
    const unsigned char* __restrict__ keys, int64_t lane_stride_b, int row_b, int d, double* __restrict__ scratch,
    int32_t* __restrict__ sel_tok, double* __restrict__ sel_score, int64_t sel_stride, int32_t* __restrict__ n_sel,
    int32_t* __restrict__ run_start, int32_t* __restrict__ run_len, int64_t run_stride, int32_t* __restrict__ n_runs, int kvg, int tkg,
    float* __restrict__ hint) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    __shared__ S3Shared S;
    __shared__ long long w_sel[(NT / 32)];
    __shared__ int band_pos[S3_BAND_CAP];
    uint32_t* lkey = reinterpret_cast<uint32_t*>(dyn_smem);
    int32_t* lpos = reinterpret_cast<int32_t*>(dyn_smem + (size_t)S3_LIST_CAP * 4);  // merged path only
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t li = blockIdx.x;
    const int64_t n = n_cand[li];
    const int64_t kk = kvt::imin(k, n);
    const float* sc = cs32 + li * cand_stride;
    const int32_t* tk = ctok + (li - (int64_t)(blockIdx.x % (unsigned)tkg)) * cand_stride;  // GQA union: one id row per group
    const QT* ql = q + li * d;
    const unsigned char* kl = keys + (li / kvg) * lane_stride_b;
    int32_t* otok = sel_tok + li * sel_stride;
    double* osc = sel_score + li * sel_stride;
    const bool vec = ((uintptr_t)sc % 16) == 0 && ((uintptr_t)tk % 16) == 0;
    if (kk <= 0) {
        if (tid == 0) { n_sel[li] = 0; if (run_start) n_runs[li] = 0; }
        return;
    }
    const double E = rec[li * 4 + 3] > 0.0 ? rec[li * 4 + 3] : rec[li * 4 + 0];  // K4-i4mma bound if set
    const double lo = rec[li * 4 + 1] - 2.0 * E;
    const double hi = rec[li * 4 + 2] + 2.0 * E;
    const double inv = hi > lo ? (double)S3_BINS / (hi - lo) : 0.0;
    const float lo_f = (float)lo, inv_f = (float)inv;
    const int n32 = (int)n;
    s3_mark(0);

    // Hint (state carried across decode steps): the bucket coordinate of the lane's previous
    // k-th estimate.  Its bucket stands in for the histogram's when the band is narrow: the merged pass below
    // then also counts the elements above the bucket, and the hint is taken only if the k-th
    // element really lies in that bucket; otherwise the histogram pass runs after all.
    const bool narrow = 2.0 * E * inv <= 0.5;
    int bstar = -1;
    long long above = 0;
    bool hinted = false;
    // A hint that missed backs off for 63 steps (stored as -63 .. -1): fresh, uncorrelated
    // queries every step pay the wasted pass once in 64 steps.
    const float hv_in = hint ? hint[li] : NAN;
    bool hint_missed = false;
    if (hint && narrow) {
        const float hv = hv_in;  // bucket coordinate of the previous k-th estimate
        if (isfinite(hv) && hv >= 1.f && hv < (float)(S3_BINS - 1)) {
            hinted = true;
            bstar = (int)hv;
        }
    }
    bool fallback = false, merged = false;
    int bsel = -1;  // the k-th element's bucket (== bstar unless a hint was one bucket off)
    double hb = 0.0, lb = 0.0;
    const WarpRange4<NT / 32> wr(n, warp);
    long long nsure = 0;
    unsigned int nband_total = 0;
    __shared__ unsigned int w_list_sure[(NT / 32)];  // 32-bit: native shared atomics (64-bit ones are CAS loops)
    __shared__ unsigned int s_cnt[5];
    int LR = hinted ? 2 : 1;
    for (;;) {
    LR = hinted ? 2 : 1;
    if (!hinted) {
    // ---- 1. bucket histogram of the estimates (4 per thread per iteration) ----
    for (int i = tid; i < S3_BINS; i += NT) S.hist[i] = 0;
    if (tid == 0) { S.list_n = 0; S.bstar = -1; S.above = 0; S.remaining = 0; }
    __syncthreads();
    // passes over the estimates batch S3_UB float4 loads per thread (memory-level parallelism)
    for (int base = 0; base < n32; base += S3_UB * 4 * NT) {
        float v[S3_UB][4];
#pragma unroll
        for (int u = 0; u < S3_UB; ++u) load4s(sc, base + (u * NT + tid) * 4, n32, vec, v[u]);
#pragma unroll
        for (int u = 0; u < S3_UB; ++u) {
            const int i = base + (u * NT + tid) * 4;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int bkt = i + e < n32 ? s3_bucket(v[u][e], lo_f, inv_f) : -1;
                if (bkt >= 0) atomicAdd(&S.hist[bkt], 1u);
            }
        }
    }
    __syncthreads();
    s3_mark(1);
    s3_find_bin<NT>(S, S.hist, S3_BINS, kk);
    s3_mark(2);
    bstar = S.bstar;
    above = S.above;
    } else {
        if (tid == 0) { S.list_n = 0; S.remaining = 0; }
        __syncthreads();
    }
    fallback = bstar < 0;
    bsel = bstar;
    nsure = 0;
    // Merged path: when the band [T - 2E, T + 2E] is narrower than half a bucket it lies in
    // buckets bstar-1..bstar+1, so ONE pass (in warp ranges) gathers those buckets' members
    // with their positions and counts the certainly-selected elements above them; T, the
    // band and the remaining sure counts then come from the short list.
    merged = !fallback && narrow;
    if (!merged) break;
        if (lane == 0) w_list_sure[warp] = 0;
        for (int base0 = wr.a; base0 < wr.b; base0 += 128 * S3_UW) {
          float vv[S3_UW][4];
#pragma unroll
          for (int u = 0; u < S3_UW; ++u) load4s(sc, base0 + 128 * u + 4 * lane, wr.b, vec, vv[u]);
          // flags of this lane's 4 x S3_UW elements as a bitmask; one warp scan + one atomic
          // per iteration place the list members (sure counts stay per lane until the end)
          // list = buckets bstar - LR .. bstar + LR (LR = 2 when hinted: the k-th may have moved
          // one bucket since the hint; 1 otherwise); the bucket offset rides in bits 29..31
          unsigned mbits = 0;
#pragma unroll
          for (int u = 0; u < S3_UW; ++u) {
            const int i = base0 + 128 * u + 4 * lane;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool in = i + e < wr.b;
                const int b = in ? s3_bucket(vv[u][e], lo_f, inv_f) : -1;
                nsure += b > bstar + LR;
                mbits |= (unsigned)(in && b >= bstar - LR && b <= bstar + LR) << (4 * u + e);
            }
          }
          const int cnt = __popc(mbits);
          const int inc = warp_incl_scan(cnt, lane);
          unsigned wb = 0;
          if (lane == 31 && inc) wb = atomicAdd(&S.list_n, (unsigned)inc);
          wb = __shfl_sync(KVT_FULL, wb, 31);
          unsigned slot = wb + (unsigned)(inc - cnt);
          while (mbits) {
            const int f = __ffs(mbits) - 1;
            mbits &= mbits - 1;
            if (slot < S3_LIST_CAP) {
                const int u = f >> 2, e = f & 3;
                const int i = base0 + 128 * u + 4 * lane + e;
                float v = vv[0][0];
#pragma unroll
                for (int uu = 0; uu < S3_UW; ++uu)
#pragma unroll
                    for (int ee = 0; ee < 4; ++ee)
                        if (uu == u && ee == e) v = vv[uu][ee];
                const uint32_t of = (uint32_t)(s3_bucket(v, lo_f, inv_f) - bstar + 2);  // 0 .. 4
                lkey[slot] = ord_key32(v);
                lpos[slot] = (int32_t)((uint32_t)i | (of << 29));
            }
            ++slot;
          }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) nsure += __shfl_xor_sync(KVT_FULL, nsure, off);
        __syncthreads();
        s3_mark(3);
        if (hinted) {
            // per-bucket counts of the list; the k-th element's bucket bt must be one of
            // bstar - 1 .. bstar + 1 (its band then stays inside the listed buckets)
            if (tid < 5) s_cnt[tid] = 0;
            if (lane == 0) w_sel[warp] = nsure;
            __syncthreads();
            const int lnh = (int)kvt::imin((long long)S.list_n, (long long)S3_LIST_CAP);
            unsigned c[5] = {0, 0, 0, 0, 0};
            for (int j = tid; j < lnh; j += NT) {
                const unsigned of = ((uint32_t)lpos[j] >> 29) & 7u;
#pragma unroll
                for (int o = 0; o < 5; ++o) c[o] += of == (unsigned)o;
            }
#pragma unroll
            for (int o = 0; o < 5; ++o)
                if (c[o]) atomicAdd(&s_cnt[o], c[o]);
            __syncthreads();
            long long ab = 0;  // elements above bucket bstar + 2
            for (int w = 0; w < (NT / 32); ++w) ab += w_sel[w];
            int bt = -1;
            if (S.list_n <= (unsigned)S3_LIST_CAP) {
                ab += s_cnt[4];  // now: above bucket bstar + 1
                for (int o = 3; o >= 1; --o) {  // bucket bstar + 1, bstar, bstar - 1
                    if (ab < kk && kk <= ab + (long long)s_cnt[o]) { bt = bstar + o - 2; break; }
                    ab += s_cnt[o];
                }
            }
            __syncthreads();  // w_sel / counters read by every thread before any reuse
            if (bt < 0) {  // the k-th element moved more than one bucket: histogram after all
                hinted = false;
                hint_missed = true;
                continue;
            }
            above = 0;  // recomputed below for bucket bt
            {
                long long a2 = 0;
                for (int w = 0; w < (NT / 32); ++w) a2 += w_sel[w];
                for (int o = 4; o > bt - bstar + 2; --o) a2 += s_cnt[o];
                above = a2;
            }
            bsel = bt;
        }
        break;
    }
    const long long need_in_bucket = kk - above;
    float hint_out = NAN;  // this step's k-th estimate: the next step's hint (merged path only)
    if (merged) {
        const int ln = (int)S.list_n;
        if (ln > S3_LIST_CAP) {
            fallback = true;
        } else {
            // T = the need_in_bucket-th largest key among the bucket-bstar members: compact
            // their keys behind the list (ballot + one atomic per warp), then the bounded
            // list select (rank count for tiny lists, 8-bit radix rounds otherwise)
            uint32_t* bkey = S.hist;  // the bucket histogram is dead once bstar is known
            __shared__ unsigned int s_nb;
            if (tid == 0) s_nb = 0;
            __syncthreads();
            for (int j0 = 0; j0 < ln; j0 += NT) {
                const int j = j0 + tid;
                const bool m = j < ln && ((((uint32_t)lpos[j] >> 29) & 7u) == (uint32_t)(bsel - bstar + 2));
                const unsigned ballot = __ballot_sync(KVT_FULL, m);
                unsigned wb = 0;
                if (lane == 0 && ballot) wb = atomicAdd(&s_nb, (unsigned)__popc(ballot));
                wb = __shfl_sync(KVT_FULL, wb, 0);
                const unsigned slot = wb + __popc(ballot & ((1u << lane) - 1));
                if (m && slot < S3_BINS) bkey[slot] = lkey[j];
            }
            __syncthreads();  // every thread has read list_n before it is reset
            if (s_nb > (unsigned)S3_BINS) fallback = true;  // (block-uniform)
            const uint32_t T32m = fallback ? 0u : s3_list_select<NT>(S, bkey, (int)s_nb, need_in_bucket);
            if (tid == 0) S.list_n = 0;  // reused as the band counter
            __syncthreads();
            const double Tk = (double)key32_to_float(T32m);
            // kept as a bucket coordinate, (T - lo) / width: invariant to a rescaled query (the
            // range [tau - 2E, Umax + 2E] scales with it), so the hint survives gain changes
            if (!fallback) hint_out = (float)((Tk - lo) * inv);
            hb = Tk + 2.0 * E;
            lb = Tk - 2.0 * E;
            // sure list members counted into their owner warp's range (WarpRange4 spans of
            // `per` elements); band members appended
            const int64_t per = ((n + (NT / 32) - 1) / (NT / 32) + 127) / 128 * 128;
            for (int j = tid; j < ln; j += NT) {
                const double sv = (double)key32_to_float(lkey[j]);
                const int pj = lpos[j] & 0x1fffffff;
                if (sv > hb) {
                    const int ow = (int)kvt::imin((NT / 32) - 1, pj / per);
                    atomicAdd(&w_list_sure[ow], 1u);
                } else if (sv >= lb) {
                    const unsigned slot = atomicAdd(&S.list_n, 1u);
                    if (slot < S3_BAND_CAP) { S.band_t[slot] = tk[pj]; band_pos[slot] = pj; }
                }
            }
            __syncthreads();
            nsure += w_list_sure[warp];
        }
    }
    if (!merged && !fallback) {
    // ---- 2. gather the k-th bucket (unordered) ----
    for (int base0 = 0; base0 < n32; base0 += S3_UB * 4 * NT) {
      float vv[S3_UB][4];
#pragma unroll
      for (int u = 0; u < S3_UB; ++u) load4s(sc, base0 + (u * NT + tid) * 4, n32, vec, vv[u]);
#pragma unroll
      for (int u = 0; u < S3_UB; ++u) {
        const int i = base0 + (u * NT + tid) * 4;
        const float* v = vv[u];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool m = i + e < n32 && s3_bucket(v[e], lo_f, inv_f) == bstar;
            const unsigned ballot = __ballot_sync(KVT_FULL, m);
            unsigned wb = 0;
            if (lane == 0 && ballot) wb = atomicAdd(&S.list_n, (unsigned)__popc(ballot));
            wb = __shfl_sync(KVT_FULL, wb, 0);
            if (m) {
                const unsigned slot = wb + __popc(ballot & ((1u << lane) - 1));
                if (slot < S3_LIST_CAP) lkey[slot] = ord_key32(v[e]);
            }
        }
      }
    }
    __syncthreads();
    fallback = S.list_n > S3_LIST_CAP;
    if (!fallback) {
        const uint32_t T32 = s3_list_select<NT>(S, lkey, (int)S.list_n, need_in_bucket);
        const double Tk = (double)key32_to_float(T32);
        hb = Tk + 2.0 * E;
        lb = Tk - 2.0 * E;
        // ---- 3. per-warp sure counts + band members (appended, unordered) ----
        if (tid == 0) S.list_n = 0;  // reused as the band counter
        __syncthreads();
        for (int base0 = wr.a; base0 < wr.b; base0 += 128 * S3_UW) {
          float vv[S3_UW][4];
#pragma unroll
          for (int u = 0; u < S3_UW; ++u) load4s(sc, base0 + 128 * u + 4 * lane, wr.b, vec, vv[u]);
#pragma unroll
          for (int u = 0; u < S3_UW; ++u) {
            const int i = base0 + 128 * u + 4 * lane;
            const float* v = vv[u];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double sv = (double)v[e];
                const bool in = i + e < wr.b;
                nsure += __popc(__ballot_sync(KVT_FULL, in && sv > hb));
                const bool bd = in && sv <= hb && sv >= lb;
                const unsigned ballot = __ballot_sync(KVT_FULL, bd);
                unsigned wb = 0;
                if (lane == 0 && ballot) wb = atomicAdd(&S.list_n, (unsigned)__popc(ballot));
                wb = __shfl_sync(KVT_FULL, wb, 0);
                if (bd) {
                    const unsigned slot = wb + __popc(ballot & ((1u << lane) - 1));
                    if (slot < S3_BAND_CAP) { S.band_t[slot] = tk[i + e]; band_pos[slot] = (int)(i + e); }
                }
            }
          }
        }
    }
    }
    s3_mark(4);
    if (!fallback) {
        if (lane == 0) w_sel[warp] = nsure;
        __syncthreads();
        nband_total = S.list_n;
        long long tot_sure = 0;
        for (int w = 0; w < (NT / 32); ++w) tot_sure += w_sel[w];
        const long long need = kk - tot_sure;
        if (nband_total > (unsigned)S3_BAND_CAP) {
            fallback = true;
        } else {
            for (int j = warp; j < (int)nband_total; j += (NT / 32)) {
                const double c = s3_canon<QT, T>(ql, kl + (int64_t)S.band_t[j] * row_b, d, lane);
                if (lane == 0) S.band_c[j] = c;
            }
            __syncthreads();
            for (int j = tid; j < (int)nband_total; j += NT) {
                const double cj = S.band_c[j];
                const int tj = S.band_t[j];
                long long better = 0;
                for (int f = 0; f < (int)nband_total; ++f) {
                    const double cf = S.band_c[f];
                    better += (cf > cj) || (cf == cj && S.band_t[f] < tj);
                }
                S.band_sel[j] = better < need ? 1 : 0;
            }
            __syncthreads();
        }
    }
    __syncthreads();
    s3_mark(5);
    if (hint && tid == 0)
        hint[li] = hint_missed ? -63.f : (hv_in < -1.5f ? hv_in + 1.f : (fallback ? NAN : hint_out));
    if (!fallback) {
        // ---- 4. stable compaction: per-warp offsets, lane-level scan inside each window ----
        long long extra = 0;  // selected band members inside this warp's range
        for (int j = lane; j < (int)nband_total; j += 32)
            extra += (band_pos[j] >= wr.a && band_pos[j] < wr.b) ? S.band_sel[j] : 0;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) extra += __shfl_xor_sync(KVT_FULL, extra, off);
        __syncthreads();
        if (lane == 0) w_sel[warp] = nsure + extra;
        __syncthreads();
        long long pos = 0;
        for (int w = 0; w < warp; ++w) pos += w_sel[w];
        // run heads from the candidate stream (tokens ascending): a selected element is a head
        // unless its stream predecessor is selected and holds the previous token.  Flags go to
        // shared memory by output position (the list area is free now).
        unsigned char* hflag = dyn_smem;
        const bool runs_fused = run_start != nullptr && kk <= (int64_t)S3_LIST_CAP * 8;
        bool carry_m = false;
        int carry_t = 0;
        if (wr.a > 0 && wr.a < wr.b) {
            const double sv = (double)sc[wr.a - 1];
            carry_t = tk[wr.a - 1];
            if (sv > hb) carry_m = true;
            else if (sv >= lb)
                for (int j = 0; j < (int)nband_total; ++j)
                    if (band_pos[j] == (int)(wr.a - 1)) { carry_m = S.band_sel[j] != 0; break; }
        }
        for (int base0 = wr.a; base0 < wr.b; base0 += 128 * S3_UWC) {
          float vv[S3_UWC][4];
          int tt[S3_UWC][4];
#pragma unroll
          for (int u = 0; u < S3_UWC; ++u) {
              const int i = base0 + 128 * u + 4 * lane;
              load4s(sc, i, wr.b, vec, vv[u]);
              if (vec && i + 4 <= wr.b) {
                  const int4 x = *reinterpret_cast<const int4*>(tk + i);
                  tt[u][0] = x.x; tt[u][1] = x.y; tt[u][2] = x.z; tt[u][3] = x.w;
              } else {
#pragma unroll
                  for (int e = 0; e < 4; ++e) tt[u][e] = i + e < wr.b ? tk[i + e] : 0;
              }
          }
#pragma unroll
          for (int u = 0; u < S3_UWC; ++u) {
            const int i = base0 + 128 * u + 4 * lane;
            const float* v = vv[u];
            bool m[4];
            double scr[4];
            int cnt = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double sv = (double)v[e];
                m[e] = false;
                scr[e] = sv;
                if (i + e < wr.b) {
                    if (sv > hb) m[e] = true;
                    else if (sv >= lb) {
                        for (int j = 0; j < (int)nband_total; ++j)
                            if (band_pos[j] == (int)(i + e)) { m[e] = S.band_sel[j] != 0; scr[e] = S.band_c[j]; break; }
                    }
                }
                cnt += m[e];
            }
            const int inc = warp_incl_scan(cnt, lane);
            long long p = pos + inc - cnt;
            // predecessor of element e = 0: lane - 1's last element, or the carry
            bool pm = __shfl_up_sync(KVT_FULL, m[3], 1);
            int pt = __shfl_up_sync(KVT_FULL, tt[u][3], 1);
            if (lane == 0) { pm = carry_m; pt = carry_t; }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (m[e]) {
                    otok[p] = tt[u][e];
                    osc[p] = scr[e];
                    if (runs_fused) hflag[p] = !(pm && pt == tt[u][e] - 1);
                    ++p;
                }
                pm = m[e];
                pt = tt[u][e];
            }
            carry_m = __shfl_sync(KVT_FULL, m[3], 31);
            carry_t = __shfl_sync(KVT_FULL, tt[u][3], 31);
            pos += __shfl_sync(KVT_FULL, inc, 31);
          }
        }
        w_sel[warp] = w_sel[warp];  // (no-op: keeps the per-warp totals for the run scan below)
    } else {
        // ---- exact fallback: canonical f64 for every candidate, 64-bit radix select ----
        double* sc64 = scratch + li * cand_stride;
        for (int64_t base = (int64_t)warp * 8; base < n; base += (int64_t)(NT / 32) * 8) {
            double p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                double acc = 0.0;
                if (base + u < n) {
                    const unsigned char* row = kl + (int64_t)tk[base + u] * row_b;
                    for (int g = lane; 4 * g < d; g += 32) {
                        double vv[4];
                        RowLd<T>::load(row, g, d, vv);
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (4 * g + e < d) acc = fma((double)ql[4 * g + e], vv[e], acc);
                    }
                }
                p[u] = acc;
            }
            const double dot = tree_8tok<double>(p, lane);
            const int t = (lane >> 2) & 7;
            if ((lane & 3) == 0 && base + t < n) sc64[base + t] = dot;
        }
        __syncthreads();
        if (tid == 0) { S.prefix = 0; S.mask = 0; S.remaining = (unsigned)kk; }
        __syncthreads();
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += NT) S.rh[i] = 0;
            __syncthreads();
            const unsigned long long pf = S.prefix, mk = S.mask;
            for (int64_t base = 0; base < n; base += NT) {
                const int64_t i = base + tid;
                int dg = 256;
                if (i < n) {
                    const uint64_t key = ord_key(sc64[i]);
                    if ((key & mk) == pf) dg = (int)((key >> shift) & 0xff);
                }
                const unsigned peers = __match_any_sync(KVT_FULL, dg);
                if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&S.rh[dg], (unsigned)__popc(peers));
            }
            __syncthreads();
            if (tid < 32) {
                unsigned loc[8], ls = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) { loc[i] = S.rh[255 - 8 * lane - i]; ls += loc[i]; }
                const unsigned inc = warp_incl_scan(ls, lane), exc = inc - ls, rem = S.remaining;
            __syncwarp();  // every lane has read S.remaining before it is rewritten
                if (exc < rem && rem <= inc) {
                    unsigned run = exc;
                    for (int i = 0; i < 8; ++i) {
                        if (run + loc[i] >= rem) {
                            const int bb = 255 - 8 * lane - i;
                            S.prefix = pf | ((unsigned long long)bb << shift);
                            S.mask = mk | (0xffull << shift);
                            S.remaining = rem - run;
                            break;
                        }
                        run += loc[i];
                    }
                }
            }
            __syncthreads();
        }
        const uint64_t T64 = S.prefix;
        const long long eq_take_total = S.remaining;
        // per-warp counts of (key > T) and ties, in warp-range order
        const WarpRange<NT / 32> w1(n, warp);
        long long c_gt = 0, c_eq = 0;
        for (int64_t base = w1.a; base < w1.b; base += 32) {
            const int64_t i = base + lane;
            uint64_t key = 0;
            if (i < w1.b) key = ord_key(sc64[i]);
            c_gt += __popc(__ballot_sync(KVT_FULL, i < w1.b && key > T64));
            c_eq += __popc(__ballot_sync(KVT_FULL, i < w1.b && key == T64));
        }
        __shared__ long long w_eq[(NT / 32)], w_gt[(NT / 32)];
        if (lane == 0) { w_eq[warp] = c_eq; w_gt[warp] = c_gt; }
        __syncthreads();
        long long eq_before = 0, pos = 0;
        for (int w = 0; w < warp; ++w) {
            const long long take = max(0LL, min(w_eq[w], eq_take_total - eq_before));
            pos += w_gt[w] + take;
            eq_before += w_eq[w];
        }
        long long eq_seen = eq_before;
        for (int64_t base = w1.a; base < w1.b; base += 32) {
            const int64_t i = base + lane;
            uint64_t key = 0;
            if (i < w1.b) key = ord_key(sc64[i]);
            const bool is_eq = i < w1.b && key == T64;
            const unsigned eqb = __ballot_sync(KVT_FULL, is_eq);
            const long long my_eq = eq_seen + __popc(eqb & ((1u << lane) - 1));
            const bool m = i < w1.b && (key > T64 || (is_eq && my_eq < eq_take_total));
            const unsigned ballot = __ballot_sync(KVT_FULL, m);
            if (m) {
                const long long p = pos + __popc(ballot & ((1u << lane) - 1));
                otok[p] = tk[i];
                osc[p] = sc64[i];
            }
            pos += __popc(ballot);
            eq_seen += __popc(eqb);
        }
    }
    s3_mark(6);
    if (tid == 0) n_sel[li] = (int32_t)kk;
    if (!run_start) return;
    if (!fallback && kk <= (int64_t)S3_LIST_CAP * 8) {
        // ---- 5. runs from the head flags (shared memory): count, block prefix, write ----
        __syncthreads();
        const unsigned char* hflag = dyn_smem;
        const long long per_w = ((kk + (NT / 32) - 1) / (NT / 32) + 31) / 32 * 32;
        const long long pa = kvt::imin(kk, warp * per_w), pb = kvt::imin(kk, pa + per_w);
        long long nh = 0;
        for (long long p = pa + lane; p - lane < pb; p += 32)
            nh += __popc(__ballot_sync(KVT_FULL, p < pb && hflag[p]));
        __syncthreads();
        if (lane == 0) w_sel[warp] = nh;
        __syncthreads();
        long long r0 = 0, tot_h = 0;
        for (int w = 0; w < (NT / 32); ++w) {
            if (w < warp) r0 += w_sel[w];
            tot_h += w_sel[w];
        }
        int32_t* rs = run_start + li * run_stride;
        int32_t* rl = run_len + li * run_stride;
        const unsigned le_mask = (2u << lane) - 1u;
        // One pass: a run's length is the distance to the next head, found in the same 32-wide
        // window (ballot bits) or, for a window's last head, at the next window's first head;
        // the warp's last run ends at the next warp's first head (or k), set after a barrier.
        // Head tokens are loaded RU windows at a time (no read-after-write chains).
        constexpr int RU = 4;
        __shared__ long long w_first_hp[(NT / 32)];
        long long r = r0, r_last = -1, p_last = -1, first_hp = -1;
        for (long long p0 = pa; p0 < pb; p0 += 32 * RU) {
            bool h[RU];
            int t[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const long long p = p0 + 32 * u + lane;
                h[u] = p < pb && hflag[p];
            }
#pragma unroll
            for (int u = 0; u < RU; ++u) t[u] = h[u] ? otok[p0 + 32 * u + lane] : 0;
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const unsigned hm = __ballot_sync(KVT_FULL, h[u]);
                if (!hm) continue;  // warp-uniform
                const long long wbase = p0 + 32 * u;
                if (h[u]) {
                    const long long idx = r + __popc(hm & le_mask) - 1;
                    rs[idx] = t[u];
                    const unsigned above = hm & ~le_mask;
                    if (above) rl[idx] = (int32_t)(__ffs(above) - 1 - lane);
                }
                const long long pf = wbase + __ffs(hm) - 1;
                if (lane == 0 && r_last >= 0) rl[r_last] = (int32_t)(pf - p_last);
                if (first_hp < 0) first_hp = pf;
                p_last = wbase + 31 - __clz(hm);
                r += __popc(hm);
                r_last = r - 1;
            }
        }
        if (lane == 0) w_first_hp[warp] = first_hp;
        __syncthreads();
        if (lane == 0 && r_last >= 0) {
            long long nx = kk;
            for (int w = warp + 1; w < (NT / 32); ++w)
                if (w_first_hp[w] >= 0) { nx = w_first_hp[w]; break; }
            rl[r_last] = (int32_t)(nx - p_last);
        }
        if (tid == 0) n_runs[li] = (int32_t)tot_h;
        s3_mark(7);
        return;
    }

    // ---- 5. fused run scan (engine.py:176-183) over the k outputs, warp-cooperative ----
    // Warp w owns output positions [wa, wb); per 32-wide window a lane tests head (previous
    // token not adjacent) and tail (next token not adjacent) with coalesced loads, run
    // indices come from ballots + one block scan of the per-warp head counts.  Run starts
    // and, temporarily, head positions are written first; lengths after a barrier.
    __syncthreads();
    {
        constexpr int RU = 4;
        const long long per_w = ((kk + (NT / 32) - 1) / (NT / 32) + 31) / 32 * 32;
        const long long wa = kvt::imin(kk, warp * per_w), wb = kvt::imin(kk, wa + per_w);
        int32_t* rs = run_start + li * run_stride;
        int32_t* rl = run_len + li * run_stride;
        const unsigned le_mask = (2u << lane) - 1u;
        long long nh = 0;
        for (long long p0 = wa; p0 < wb; p0 += 32 * RU) {
            bool hd[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const long long p = p0 + 32 * u + lane;
                hd[u] = p < wb && (p == 0 || otok[p] != otok[p - 1] + 1);
            }
#pragma unroll
            for (int u = 0; u < RU; ++u) nh += __popc(__ballot_sync(KVT_FULL, hd[u]));
        }
        __syncthreads();  // w_sel is reused for the per-warp head counts
        if (lane == 0) w_sel[warp] = nh;
        __syncthreads();
        long long base_r = 0, tot_h = 0;
        for (int w = 0; w < (NT / 32); ++w) {
            if (w < warp) base_r += w_sel[w];
            tot_h += w_sel[w];
        }
        for (int pass = 0; pass < 2; ++pass) {
            long long r0 = base_r;
            for (long long p0 = wa; p0 < wb; p0 += 32 * RU) {
                int t[RU];
                bool hd[RU], tl[RU];
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const long long p = p0 + 32 * u + lane;
                    t[u] = p < wb ? otok[p] : 0;
                    hd[u] = p < wb && (p == 0 || t[u] != otok[p - 1] + 1);
                    tl[u] = p < wb && (p == kk - 1 || otok[p + 1] != t[u] + 1);
                }
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const long long p = p0 + 32 * u + lane;
                    const unsigned hm = __ballot_sync(KVT_FULL, hd[u]);
                    const long long r = r0 + __popc(hm & le_mask) - 1;  // run of position p
                    if (pass == 0 && hd[u]) { rs[r] = t[u]; rl[r] = (int32_t)p; }
                    if (pass == 1 && tl[u]) rl[r] = (int32_t)(p + 1 - rl[r]);
                    r0 += __popc(hm);
                }
            }
            __syncthreads();
        }
        if (tid == 0) n_runs[li] = (int32_t)tot_h;
    }
}

}  // namespace kvt

using namespace kvt;



template <typename QT, typename T, int NT>
static int launch_select3_nt(const float* cs32, const int32_t* ctok, const int32_t* n_cand, int64_t cand_stride,
                             const double* rec, int64_t n_lanes, int64_t k, const void* q, const void* keys,
                             int64_t ls_b, int row_b, int d, double* scratch, int32_t* sel_tok, double* sel_score,
                             int64_t sel_stride, int32_t* n_sel, int32_t* run_start, int32_t* run_len,
                             int64_t run_stride, int32_t* n_runs, cudaStream_t st) {
    const size_t smem = (size_t)S3_LIST_CAP * 8;  // list keys + positions
    KVT_PER_DEVICE(bool, configured);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(topk_select3_kernel<QT, T, NT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        configured = true;
    }
    launch_pdl(topk_select3_kernel<QT, T, NT>, dim3((unsigned)n_lanes), dim3(NT), smem, st, cs32, ctok, n_cand,
               cand_stride, rec, k, (const QT*)q, (const unsigned char*)keys, ls_b, row_b, d, scratch, sel_tok,
               sel_score, sel_stride, n_sel, run_start, run_len, run_stride, n_runs, kv_group_current(),
               cand_group_current(), sel_hint_current());
    return kvt_check_launch();
}

// Fewer lanes than SMs: 1024-thread CTAs (one per SM) split each lane's passes over 32 warps;
// otherwise 512 (two per SM).
template <typename QT, typename T>
static int launch_select3(const float* cs32, const int32_t* ctok, const int32_t* n_cand, int64_t cand_stride,
                          const double* rec, int64_t n_lanes, int64_t k, const void* q, const void* keys,
                          int64_t lane_stride, int d, double* scratch, int32_t* sel_tok, double* sel_score,
                          int64_t sel_stride, int32_t* n_sel, int32_t* run_start, int32_t* run_len,
                          int64_t run_stride, int32_t* n_runs, cudaStream_t st) {
    const int row_b = RowLd<T>::row_bytes(d);
    const int64_t ls_b = std::is_same<T, I4>::value ? lane_stride : lane_stride * (int64_t)sizeof(T);
    if (n_lanes < kvt::sm_count())
        return launch_select3_nt<QT, T, 1024>(cs32, ctok, n_cand, cand_stride, rec, n_lanes, k, q, keys, ls_b, row_b,
                                              d, scratch, sel_tok, sel_score, sel_stride, n_sel, run_start, run_len,
                                              run_stride, n_runs, st);
    return launch_select3_nt<QT, T, 512>(cs32, ctok, n_cand, cand_stride, rec, n_lanes, k, q, keys, ls_b, row_b, d,
                                         scratch, sel_tok, sel_score, sel_stride, n_sel, run_start, run_len,
                                         run_stride, n_runs, st);
}

extern "C" int kvt_debug_select_phases(unsigned long long* buf) {
    const cudaError_t e = cudaMemcpyToSymbol(g_s3_phase, &buf, sizeof(buf));
    return e == cudaSuccess ? KVT_OK : kvt_set_cuda_error(e);
}

extern "C" int kvt_topk_select_band(const float* cs32, const int32_t* ctok, const int32_t* n_cand,
                                    int64_t cand_stride, const double* rec, int64_t n_lanes, int64_t k, const void* q,
                                    int q_dtype, const void* keys, int key_dtype, int64_t lane_stride, int d,
                                    double* scratch, int32_t* sel_tok, double* sel_score, int64_t sel_stride,
                                    int32_t* n_sel, int32_t* run_start, int32_t* run_len, int64_t run_stride,
                                    int32_t* n_runs, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!cs32 || !ctok || !n_cand || !rec || !q || !keys || !scratch || !sel_tok || !sel_score || !n_sel)
        return KVT_ERR_ARG;
    if (k < 0) return KVT_ERR_K;
    if (n_lanes == 0) return KVT_OK;
    if (n_lanes > 2147483647LL) return KVT_ERR_ARG;
#define KVT_S(QT, TT) return launch_select3<QT, TT>(cs32, ctok, n_cand, cand_stride, rec, n_lanes, k, q, keys, lane_stride, d, scratch, sel_tok, sel_score, sel_stride, n_sel, run_start, run_len, run_stride, n_runs, st)
    if (q_dtype == KVT_F32) {
        switch (key_dtype) {
            case KVT_F32: KVT_S(float, float);
            case KVT_BF16: KVT_S(float, __nv_bfloat16);
            case KVT_F16: KVT_S(float, __half);
            case KVT_I4: KVT_S(float, I4);
        }
    } else if (q_dtype == KVT_F64) {
        switch (key_dtype) {
            case KVT_F32: KVT_S(double, float);
            case KVT_BF16: KVT_S(double, __nv_bfloat16);
            case KVT_F16: KVT_S(double, __half);
            case KVT_I4: KVT_S(double, I4);
        }
    }
#undef KVT_S
    return KVT_ERR_DTYPE;
}
