// select2.cu -- K5 on fast f32 scores, exact by construction; the cluster-per-lane variant
// used when there are too few lanes to fill the GPU with one CTA each (select3.cu).
//
// K4's f32 estimate s of each candidate's canonical f64 dot c satisfies |s - c| <= E, a
// rigorous per-lane bound computed by the plan (E = err_factor * max A over candidates,
// A = sum |q||k| per chunk from K3).  Let T be the exact k-th largest s (32-bit radix
// select, 4 passes).  The k-th largest canonical dot S_k lies in [T - E, T + E], so
//   s > T + 2E  =>  c > S_k            (selected, whatever the ties)
//   s < T - 2E  =>  c < S_k            (not selected)
// and only the "band" [T - 2E, T + 2E] (typically 0-3 tokens per lane) is re-scored in the
// canonical f64 order from the key rows; the band's top (k - #above) by (c desc, token asc)
// completes the set.  The result is the oracle's exact canonical top-k set.  If the band is
// wide (heavy ties, e.g. identical keys) the cluster falls back to re-scoring its whole
// slice canonically and running the 64-bit radix select of select.cu's algorithm.
// Scores written to sel_score are s for the sure tokens (|error| <= E) and c for the band
// (all tokens exact in the fallback).  One thread-block cluster (<= 8 CTAs, DSMEM) per lane,
// the K6 run scan fused at the end.
#include <cooperative_groups.h>

#include <type_traits>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace kvt {

constexpr int S2_THREADS = 512;
constexpr int S2_LIST_CAP = 4096;
constexpr int S2_BAND_CAP = 256;        // band members per CTA
constexpr int S2_BAND_TOTAL_CAP = 1024; // per lane

struct S2Shared {
    unsigned short list[S2_LIST_CAP];
    double band_c[S2_BAND_CAP];
    int band_t[S2_BAND_CAP];
    unsigned char band_sel[S2_BAND_CAP];
    unsigned int hist[2][256];
    unsigned int tot[256];
    long long scan_sh[33];
    unsigned long long prefix, mask;
    unsigned int list_n;
    int list_ok;
    unsigned int remaining;
    int done;
    // per-CTA counts published to the cluster
    unsigned int cnt_a, cnt_b, cnt_heads;
    unsigned int band_n;
};

// One radix pass over the staged keys (u32 or u64), 8-bit digit at `shift`, with the
// histogram summed across the cluster through DSMEM; updates S.prefix/mask/remaining.
template <typename K>
__device__ __forceinline__ void radix_pass(cg::cluster_group& cluster, S2Shared& S, const K* keys, int64_t cnt,
                                           int shift, int buf, bool allow_done) {
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned CL = cluster.num_blocks();
    unsigned int* h = S.hist[buf];
    for (int i = tid; i < 256; i += S2_THREADS) h[i] = 0;
    __syncthreads();
    const unsigned long long prefix = S.prefix, mask = S.mask;
    const bool use_list = S.list_ok;
    const int64_t span = use_list ? (int64_t)S.list_n : cnt;
    for (int64_t base = 0; base < span; base += S2_THREADS) {
        const int64_t j = base + tid;
        int digit = 256;
        if (j < span) {
            const int64_t i = use_list ? (int64_t)S.list[j] : j;
            const unsigned long long key = (unsigned long long)keys[i];
            if ((key & mask) == prefix) digit = (int)((key >> shift) & 0xff);
        }
        const unsigned peers = __match_any_sync(KVT_FULL, digit);
        if (digit < 256 && lane == __ffs(peers) - 1) atomicAdd(&h[digit], (unsigned)__popc(peers));
    }
    cluster.sync();
    for (int b = tid; b < 256; b += S2_THREADS) {
        unsigned int acc = 0;
        for (unsigned r = 0; r < CL; ++r) acc += cluster.map_shared_rank(S.hist[buf], r)[b];
        S.tot[b] = acc;
    }
    __syncthreads();
    if (tid < 32) {
        unsigned int loc[8];
        unsigned int lsum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            loc[i] = S.tot[255 - 8 * lane - i];
            lsum += loc[i];
        }
        const unsigned int inc = warp_incl_scan(lsum, lane);
        const unsigned int exc = inc - lsum;
        const unsigned int rem = S.remaining;
        __syncwarp();  // every lane has read S.remaining before it is rewritten
        if (exc < rem && rem <= inc) {
            unsigned int run = exc;
            for (int i = 0; i < 8; ++i) {
                if (run + loc[i] >= rem) {
                    const int b = 255 - 8 * lane - i;
                    S.prefix = prefix | ((unsigned long long)b << shift);
                    S.mask = mask | (0xffull << shift);
                    S.remaining = rem - run;
                    if (allow_done && loc[i] == rem - run) S.done = 1;
                    break;
                }
                run += loc[i];
            }
        }
    }
    __syncthreads();
}

// After a pass, gather the members of the current bucket (indices into the slice).
template <typename K>
__device__ __forceinline__ void build_list(S2Shared& S, const K* keys, int64_t cnt) {
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) S.list_n = 0;
    __syncthreads();
    const unsigned long long pf = S.prefix, mk = S.mask;
    for (int64_t base = 0; base < cnt; base += S2_THREADS) {
        const int64_t i = base + tid;
        const bool m = i < cnt && (((unsigned long long)keys[i]) & mk) == pf;
        const unsigned ballot = __ballot_sync(KVT_FULL, m);
        unsigned wbase = 0;
        if (lane == 0 && ballot) wbase = atomicAdd(&S.list_n, (unsigned)__popc(ballot));
        wbase = __shfl_sync(KVT_FULL, wbase, 0);
        if (m) {
            const unsigned slot = wbase + __popc(ballot & ((1u << lane) - 1));
            if (slot < S2_LIST_CAP) S.list[slot] = (unsigned short)i;
        }
    }
    __syncthreads();
    if (tid == 0) S.list_ok = (S.list_n <= S2_LIST_CAP) && cnt <= 65535;
    __syncthreads();
}

// Canonical f64 dot of one key row with q, by one warp (lane l owns dims 4l..4l+3 (+128r)).
template <typename QT, typename T>
__device__ __forceinline__ double warp_canon_dot(const QT* q, const unsigned char* row, int d, int lane) {
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

template <typename QT, typename T>
__global__ void __launch_bounds__(S2_THREADS) topk_select2_kernel(
    const float* __restrict__ cs32, const int32_t* __restrict__ ctok, const int32_t* __restrict__ n_cand,
    int64_t cand_stride, const double* __restrict__ err, int64_t k, const QT* __restrict__ q,
    const unsigned char* __restrict__ keys, int64_t lane_stride_b, int row_b, int d, int32_t* __restrict__ sel_tok,
    double* __restrict__ sel_score, int64_t sel_stride, int32_t* __restrict__ n_sel, int slice_cap,
    int32_t* __restrict__ run_start, int32_t* __restrict__ run_len, int64_t run_stride, int32_t* __restrict__ n_runs, int kvg, int tkg) {
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    __shared__ S2Shared S;
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const unsigned CL = cluster.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t li = blockIdx.y;
    const int64_t n = n_cand[li];
    const int64_t kk = kvt::imin(k, n);
    const int64_t slice = (n + CL - 1) / CL;
    const int64_t lo = kvt::imin(n, (int64_t)rank * slice);
    const int64_t cnt = kvt::imin(n, lo + slice) - lo;
    const float* sc = cs32 + li * cand_stride + lo;
    const int32_t* tk = ctok + (li / tkg) * tkg * cand_stride + lo;  // GQA union: one id row per group
    const QT* ql = q + li * d;
    const unsigned char* kl = keys + (li / kvg) * lane_stride_b;
    uint32_t* k32 = reinterpret_cast<uint32_t*>(dyn_smem);
    uint64_t* k64 = reinterpret_cast<uint64_t*>(dyn_smem);
    // cnt <= slice_cap is guaranteed by the host (cluster size chosen from cand_stride)

    for (int64_t i = tid; i < cnt; i += S2_THREADS) k32[i] = ord_key32(sc[i]);
    if (tid == 0) {
        S.prefix = 0; S.mask = 0; S.remaining = (unsigned)kk; S.done = (kk <= 0);
        S.list_ok = 0; S.list_n = 0;
    }
    __syncthreads();

    // per-thread contiguous range of the slice (stable order for the compactions)
    const int64_t per = (cnt + S2_THREADS - 1) / S2_THREADS;
    const int64_t a = kvt::imin(cnt, tid * per), b = kvt::imin(cnt, a + per);

    bool fallback = false;
    double hi = 0.0, lo_ = 0.0;
    long long need = 0;
    if (kk > 0) {
        // ---- exact k-th largest f32 estimate: 4 passes over 32-bit keys ----
        int buf = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
            radix_pass<uint32_t>(cluster, S, k32, cnt, shift, buf, false);
            buf ^= 1;
            if (shift == 16) build_list<uint32_t>(S, k32, cnt);
        }
        const double Tk = (double)key32_to_float((uint32_t)S.prefix);
        const double E = err[li * 4 + 3] > 0.0 ? err[li * 4 + 3] : err[li * 4];  // [E, tau, Umax, E_i4mma]
        hi = Tk + 2.0 * E;
        lo_ = Tk - 2.0 * E;
        // ---- count sure tokens and the band ----
        long long nhi = 0, nband = 0;
        for (int64_t i = a; i < b; ++i) {
            const double s = (double)sc[i];
            nhi += s > hi;
            nband += (s >= lo_ && s <= hi);
        }
        long long tot_hi, tot_band;
        block_excl_scan<long long>(nhi, S.scan_sh, tot_hi);
        const long long ex_band = block_excl_scan<long long>(nband, S.scan_sh, tot_band);
        if (tid == 0) { S.cnt_a = (unsigned)tot_hi; S.cnt_b = (unsigned)tot_band; }
        cluster.sync();
        long long all_hi = 0, all_band = 0, max_band = 0;
        for (unsigned r = 0; r < CL; ++r) {
            const S2Shared* rs = cluster.map_shared_rank(&S, r);
            all_hi += rs->cnt_a;
            all_band += rs->cnt_b;
            max_band = max(max_band, (long long)rs->cnt_b);
        }
        need = kk - all_hi;
        fallback = all_band > S2_BAND_TOTAL_CAP || max_band > S2_BAND_CAP;
        if (!fallback) {
            // ---- re-score the band canonically (f64) ----
            long long pos = ex_band;
            for (int64_t i = a; i < b; ++i) {
                const double s = (double)sc[i];
                if (s >= lo_ && s <= hi) S.band_t[pos++] = tk[i];
            }
            if (tid == 0) S.band_n = (unsigned)tot_band;
            __syncthreads();
            for (int j = warp; j < (int)tot_band; j += S2_THREADS / 32) {
                const double c = warp_canon_dot<QT, T>(ql, kl + (int64_t)S.band_t[j] * row_b, d, lane);
                if (lane == 0) S.band_c[j] = c;
            }
            cluster.sync();
            // rank of each local band member among all band members: (c desc, token asc)
            for (int j = tid; j < (int)tot_band; j += S2_THREADS) {
                const double cj = S.band_c[j];
                const int tj = S.band_t[j];
                long long better = 0;
                for (unsigned r = 0; r < CL; ++r) {
                    const S2Shared* rs = cluster.map_shared_rank(&S, r);
                    const int nb = (int)rs->band_n;
                    for (int f = 0; f < nb; ++f) {
                        const double cf = rs->band_c[f];
                        better += (cf > cj) || (cf == cj && rs->band_t[f] < tj);
                    }
                }
                S.band_sel[j] = better < need ? 1 : 0;
            }
            __syncthreads();
        } else {
            // ---- wide band (ties): canonical f64 for the whole slice, 64-bit radix select ----
            for (int64_t base = (int64_t)warp * 8; base < cnt; base += (int64_t)(S2_THREADS / 32) * 8) {
                double p[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    double acc = 0.0;
                    if (base + u < cnt) {
                        const unsigned char* row = kl + (int64_t)tk[base + u] * row_b;
                        for (int g = lane; 4 * g < d; g += 32) {
                            double v[4];
                            RowLd<T>::load(row, g, d, v);
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (4 * g + e < d) acc = fma((double)ql[4 * g + e], v[e], acc);
                        }
                    }
                    p[u] = acc;
                }
                const double dot = tree_8tok<double>(p, lane);
                const int t = (lane >> 2) & 7;
                if ((lane & 3) == 0 && base + t < cnt) k64[base + t] = ord_key(dot);
            }
            if (tid == 0) {
                S.prefix = 0; S.mask = 0; S.remaining = (unsigned)kk; S.done = 0;
                S.list_ok = 0; S.list_n = 0;
            }
            cluster.sync();
            int buf = 0;
            for (int shift = 56; shift >= 0; shift -= 8) {
                if (S.done) break;
                radix_pass<uint64_t>(cluster, S, k64, cnt, shift, buf, true);
                buf ^= 1;
                if (shift == 40 && !S.done) build_list<uint64_t>(S, k64, cnt);
            }
        }
    }

    // ---- compaction (ascending token order) ----
    const unsigned long long prefix = S.prefix, mask = S.mask;
    const unsigned int remaining = S.remaining;
    long long n_a = 0, n_b = 0;  // fast: selected count | fallback: gt, eq
    if (kk > 0) {
        if (!fallback) {
            long long bp = 0;
            {
                // band members before this thread's range (same order as the band list)
                long long nb = 0;
                for (int64_t i = a; i < b; ++i) { const double s = sc[i]; nb += (s >= lo_ && s <= hi); }
                long long tot;
                bp = block_excl_scan<long long>(nb, S.scan_sh, tot);
            }
            long long bpp = bp;
            for (int64_t i = a; i < b; ++i) {
                const double s = (double)sc[i];
                if (s > hi) ++n_a;
                else if (s >= lo_) n_a += S.band_sel[bpp++];
            }
        } else {
            for (int64_t i = a; i < b; ++i) {
                const unsigned long long km = k64[i] & mask;
                n_a += km > prefix;
                n_b += km == prefix;
            }
        }
    }
    long long tot_a, tot_b;
    const long long ex_a = block_excl_scan<long long>(n_a, S.scan_sh, tot_a);
    const long long ex_b = block_excl_scan<long long>(n_b, S.scan_sh, tot_b);
    if (tid == 0) { S.cnt_a = (unsigned)tot_a; S.cnt_b = (unsigned)tot_b; }
    cluster.sync();
    long long out_base = 0, eq_before = 0;
    for (unsigned r = 0; r < rank; ++r) {
        const S2Shared* rs = cluster.map_shared_rank(&S, r);
        const long long g = rs->cnt_a, e = rs->cnt_b;
        if (!fallback) out_base += g;
        else {
            out_base += g + max(0LL, min(e, (long long)remaining - eq_before));
            eq_before += e;
        }
    }
    const long long eq_take = fallback ? max(0LL, min(tot_b, (long long)remaining - eq_before)) : 0;
    int32_t* otok = sel_tok + li * sel_stride;
    double* osc = sel_score + li * sel_stride;
    long long p0 = 0, p1 = 0;
    if (kk > 0) {
        if (!fallback) {
            long long bp;
            {
                long long nb = 0;
                for (int64_t i = a; i < b; ++i) { const double s = sc[i]; nb += (s >= lo_ && s <= hi); }
                long long tot;
                bp = block_excl_scan<long long>(nb, S.scan_sh, tot);
            }
            long long pos = out_base + ex_a;
            p0 = pos;
            for (int64_t i = a; i < b; ++i) {
                const double s = (double)sc[i];
                if (s > hi) { otok[pos] = tk[i]; osc[pos] = s; ++pos; }
                else if (s >= lo_) {
                    if (S.band_sel[bp]) { otok[pos] = tk[i]; osc[pos] = S.band_c[bp]; ++pos; }
                    ++bp;
                }
            }
            p1 = pos;
        } else {
            long long pos = out_base + ex_a + min(ex_b, eq_take);
            p0 = pos;
            long long eq_seen = ex_b;
            for (int64_t i = a; i < b; ++i) {
                const unsigned long long key = k64[i];
                const unsigned long long km = key & mask;
                bool take = false;
                if (km > prefix) take = true;
                else if (km == prefix) { take = eq_seen < eq_take; ++eq_seen; }
                if (take) { otok[pos] = tk[i]; osc[pos] = key_to_double(key); ++pos; }
            }
            p1 = pos;
        }
    } else {
        // keep the block scans balanced (all threads took part above)
    }
    if (rank == 0 && tid == 0) n_sel[li] = (int32_t)kk;

    if (run_start && kk > 0) {
        // ---- fused K6 (engine.py:176-183) ----
        cluster.sync();
        long long heads = 0;
        for (long long p = p0; p < p1; ++p) heads += (p == 0 || otok[p] != otok[p - 1] + 1);
        long long tot_h;
        const long long ex_h = block_excl_scan<long long>(heads, S.scan_sh, tot_h);
        if (tid == 0) S.cnt_heads = (unsigned)tot_h;
        cluster.sync();
        long long run_base = 0, all_runs = 0;
        for (unsigned r = 0; r < CL; ++r) {
            const long long h = cluster.map_shared_rank(&S, r)->cnt_heads;
            if (r < rank) run_base += h;
            all_runs += h;
        }
        int32_t* rs = run_start + li * run_stride;
        int32_t* rl = run_len + li * run_stride;
        long long ridx = run_base + ex_h - 1;
        for (long long p = p0; p < p1; ++p) {
            if (p == 0 || otok[p] != otok[p - 1] + 1) {
                ++ridx;
                rs[ridx] = otok[p];
                rl[ridx] = (int32_t)p;
            }
        }
        cluster.sync();
        ridx = run_base + ex_h - 1;
        for (long long p = p0; p < p1; ++p) {
            if (p == 0 || otok[p] != otok[p - 1] + 1) ++ridx;
            if (p == kk - 1 || otok[p + 1] != otok[p] + 1) rl[ridx] = (int32_t)(p + 1 - rl[ridx]);
        }
        if (rank == 0 && tid == 0) n_runs[li] = (int32_t)all_runs;
    } else if (run_start && rank == 0 && tid == 0) {
        n_runs[li] = 0;
    }
    cluster.sync();  // keep shared memory alive until every DSMEM read in the cluster is done
}

}  // namespace kvt

using namespace kvt;

constexpr int S2_SLICE_CAP = 20480;  // u64 keys of the fallback (160 KB)

template <typename QT, typename T>
static int launch_select2(const float* cs32, const int32_t* ctok, const int32_t* n_cand, int64_t cand_stride,
                          const double* err, int64_t n_lanes, int64_t k, const void* q, const void* keys,
                          int64_t lane_stride, int d, int32_t* sel_tok, double* sel_score, int64_t sel_stride,
                          int32_t* n_sel, int32_t* run_start, int32_t* run_len, int64_t run_stride, int32_t* n_runs,
                          cudaStream_t st) {
    const int row_b = RowLd<T>::row_bytes(d);
    const int64_t ls_b = std::is_same<T, I4>::value ? lane_stride : lane_stride * (int64_t)sizeof(T);
    int CL = (int)kvt::imin(8, kvt::imax(1, (cand_stride + 4095) / 4096));
    const int64_t slice = (cand_stride + CL - 1) / CL;
    if (slice > S2_SLICE_CAP) return KVT_ERR_SHAPE;
    const size_t smem = (size_t)slice * sizeof(uint64_t);
    KVT_PER_DEVICE(bool, configured);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(topk_select2_kernel<QT, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             S2_SLICE_CAP * (int)sizeof(uint64_t));
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, (unsigned)n_lanes, 1);
    cfg.blockDim = dim3(S2_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, topk_select2_kernel<QT, T>, cs32, ctok, n_cand, cand_stride, err, k,
                                       (const QT*)q, (const unsigned char*)keys, ls_b, row_b, d, sel_tok, sel_score,
                                       sel_stride, n_sel, (int)slice, run_start, run_len, run_stride, n_runs,
                                       kv_group_current(), cand_group_current());
    if (e != cudaSuccess) return kvt_set_cuda_error(e);
    return kvt_check_launch();
}

int kvt_topk_select_band_cluster(const float* cs32, const int32_t* ctok, const int32_t* n_cand, int64_t cand_stride,
                         const double* err, int64_t n_lanes, int64_t k, const void* q, int q_dtype, const void* keys,
                         int key_dtype, int64_t lane_stride, int d, int32_t* sel_tok, double* sel_score,
                         int64_t sel_stride, int32_t* n_sel, int32_t* run_start, int32_t* run_len, int64_t run_stride,
                         int32_t* n_runs, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!cs32 || !ctok || !n_cand || !err || !q || !keys || !sel_tok || !sel_score || !n_sel) return KVT_ERR_ARG;
    if (k < 0) return KVT_ERR_K;
    if (n_lanes == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
#define KVT_S(QT, TT) return launch_select2<QT, TT>(cs32, ctok, n_cand, cand_stride, err, n_lanes, k, q, keys, lane_stride, d, sel_tok, sel_score, sel_stride, n_sel, run_start, run_len, run_stride, n_runs, st)
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
