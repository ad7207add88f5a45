// select.cu -- K5 exact top-k (score desc, token asc) over the candidate logits.
//
// Result contract of chunk_tree.py:233-338 select_top_k (== brute force lexsort,
// engine.py:337-339).  One thread-block CLUSTER per lane (up to 8 CTAs on one GPC): each
// CTA stages a contiguous slice of the lane's candidates (as orderable u64 keys) in shared
// memory, then 8 radix passes of 8 bits find the exact k-th key T.  Per pass every CTA
// builds a 256-bin histogram of its slice (warp-aggregated smem atomics), the histograms
// are summed through distributed shared memory (DSMEM), and every CTA derives the same
// digit.  Histograms are double-buffered so one cluster barrier per pass suffices.  The
// final compaction keeps key > T plus the lowest-index (k - #gt) keys == T; slices are in
// ascending token order, so a cluster-wide exclusive scan of per-CTA counts gives each
// CTA its output offset and the result comes out sorted by token.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace kvt {

constexpr int SEL_THREADS = 512;
constexpr int SEL_MAX_CLUSTER = 8;

constexpr int SEL_LIST_CAP = 4096;  // survivors of the first 3 passes, scanned instead of the slice

struct SelShared {
    unsigned short list[SEL_LIST_CAP];
    unsigned int list_n;
    int list_ok;
    unsigned int hist[2][256];
    unsigned int tot[256];
    unsigned int cnt_gt, cnt_eq, cnt_heads;  // per-CTA counts published to the cluster
    long long scan_sh[33];
    unsigned long long prefix, mask;
    unsigned int remaining;
    int done;
};

__global__ void __launch_bounds__(SEL_THREADS) topk_select_kernel(
    const double* __restrict__ cand_score, const int32_t* __restrict__ cand_tok, const int32_t* __restrict__ n_cand,
    int64_t cand_stride, int64_t k, int32_t* __restrict__ sel_tok, double* __restrict__ sel_score, int64_t sel_stride,
    int32_t* __restrict__ n_sel, int slice_cap, int32_t* __restrict__ run_start, int32_t* __restrict__ run_len,
    int64_t run_stride, int32_t* __restrict__ n_runs) {
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    __shared__ SelShared S;
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const unsigned CL = cluster.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t li = blockIdx.y;
    const int64_t n = n_cand[li];
    const int64_t kk = kvt::imin(k, n);
    const int64_t slice = (n + CL - 1) / CL;
    const int64_t lo = kvt::imin(n, (int64_t)rank * slice);
    const int64_t hi = kvt::imin(n, lo + slice);
    const int64_t cnt = hi - lo;
    const double* sc = cand_score + li * cand_stride + lo;
    const bool staged = cnt <= slice_cap;
    uint64_t* keys = reinterpret_cast<uint64_t*>(dyn_smem);

    if (staged)
        for (int64_t i = tid; i < cnt; i += SEL_THREADS) keys[i] = ord_key(sc[i]);
    if (tid == 0) { S.prefix = 0; S.mask = 0; S.remaining = (unsigned)kk; S.done = (kk <= 0); S.list_ok = 0; S.list_n = 0; }
    __syncthreads();

    auto key_at = [&](int64_t i) -> uint64_t { return staged ? keys[i] : ord_key(sc[i]); };

    int buf = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        if (S.done) break;  // uniform across the cluster (derived from identical data)
        unsigned int* h = S.hist[buf];
        for (int i = tid; i < 256; i += SEL_THREADS) h[i] = 0;
        __syncthreads();
        const unsigned long long prefix = S.prefix, mask = S.mask;
        const bool use_list = S.list_ok;
        const int64_t span = use_list ? (int64_t)S.list_n : cnt;
        for (int64_t base = 0; base < span; base += SEL_THREADS) {
            const int64_t j = base + tid;
            int digit = 256;
            if (j < span) {
                const int64_t i = use_list ? (int64_t)S.list[j] : j;
                const uint64_t key = key_at(i);
                if ((key & mask) == prefix) digit = (int)((key >> shift) & 0xff);
            }
            const unsigned peers = __match_any_sync(KVT_FULL, digit);
            if (digit < 256 && lane == __ffs(peers) - 1) atomicAdd(&h[digit], (unsigned)__popc(peers));
        }
        cluster.sync();
        // every CTA sums all CTAs' histograms (DSMEM): one bin per thread, CL remote loads each
        for (int b = tid; b < 256; b += SEL_THREADS) {
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
            if (exc < rem && rem <= inc) {
                unsigned int run = exc;
                for (int i = 0; i < 8; ++i) {
                    if (run + loc[i] >= rem) {
                        const int b = 255 - 8 * lane - i;
                        S.prefix = prefix | ((unsigned long long)b << shift);
                        S.mask = mask | (0xffull << shift);
                        S.remaining = rem - run;
                        // the whole bucket is taken: no further passes needed
                        if (loc[i] == rem - run) S.done = 1;
                        break;
                    }
                    run += loc[i];
                }
            }
        }
        __syncthreads();
        buf ^= 1;
        // after the 3rd pass the surviving bucket is small: gather its members once
        if (shift == 40 && !S.done && staged && cnt <= 65535) {
            const unsigned long long pf = S.prefix, mk = S.mask;
            for (int64_t base = 0; base < cnt; base += SEL_THREADS) {
                const int64_t i = base + tid;
                const bool m = i < cnt && (keys[i] & mk) == pf;
                const unsigned ballot = __ballot_sync(KVT_FULL, m);
                unsigned wbase = 0;
                if (lane == 0 && ballot) wbase = atomicAdd(&S.list_n, (unsigned)__popc(ballot));
                wbase = __shfl_sync(KVT_FULL, wbase, 0);
                if (m) {
                    const unsigned slot = wbase + __popc(ballot & ((1u << lane) - 1));
                    if (slot < SEL_LIST_CAP) S.list[slot] = (unsigned short)i;
                }
            }
            __syncthreads();
            if (tid == 0) S.list_ok = S.list_n <= SEL_LIST_CAP;
            __syncthreads();
        }
    }

    // ---- compaction: key&mask > prefix, or == prefix and among the first `remaining` ----
    const unsigned long long prefix = S.prefix, mask = S.mask;
    const unsigned int remaining = S.remaining;
    const bool any = kk > 0;
    // each thread owns a contiguous run of the slice (stable order)
    const int64_t per = (cnt + SEL_THREADS - 1) / SEL_THREADS;
    const int64_t a = kvt::imin(cnt, tid * per), b = kvt::imin(cnt, a + per);
    long long ngt = 0, neq = 0;
    if (any)
        for (int64_t i = a; i < b; ++i) {
            const uint64_t km = key_at(i) & mask;
            ngt += km > prefix;
            neq += km == prefix;
        }
    long long tot_gt, tot_eq;
    const long long ex_gt = block_excl_scan<long long>(ngt, S.scan_sh, tot_gt);
    const long long ex_eq = block_excl_scan<long long>(neq, S.scan_sh, tot_eq);
    if (tid == 0) { S.cnt_gt = (unsigned)tot_gt; S.cnt_eq = (unsigned)tot_eq; }
    cluster.sync();
    long long out_base = 0, eq_before = 0;
    for (unsigned r = 0; r < rank; ++r) {
        const SelShared* rs = cluster.map_shared_rank(&S, r);
        const long long g = rs->cnt_gt, e = rs->cnt_eq;
        const long long take = max(0LL, min(e, (long long)remaining - eq_before));
        out_base += g + take;
        eq_before += e;
    }
    const long long eq_take = max(0LL, min(tot_eq, (long long)remaining - eq_before));
    if (any) {
        int32_t* otok = sel_tok + li * sel_stride;
        double* osc = sel_score + li * sel_stride;
        const int32_t* tk = cand_tok + li * cand_stride + lo;
        long long pos = out_base + ex_gt + min(ex_eq, eq_take);
        long long eq_seen = ex_eq;
        for (int64_t i = a; i < b; ++i) {
            const uint64_t km = key_at(i) & mask;
            bool take = false;
            if (km > prefix) take = true;
            else if (km == prefix) { take = eq_seen < eq_take; ++eq_seen; }
            if (take) {
                otok[pos] = tk[i];
                osc[pos] = sc[i];
                ++pos;
            }
        }
    }
    if (rank == 0 && tid == 0) n_sel[li] = (int32_t)kk;
    if (run_start && any) {
        // ---- fused K6: runs of consecutive selected tokens (engine.py:176-183) ----
        // this thread's output positions are [p0, p1) (its selected elements, in order)
        int32_t* otok = sel_tok + li * sel_stride;
        const long long p0 = out_base + ex_gt + min(ex_eq, eq_take);
        long long taken_eq = max(0LL, min(ex_eq + neq, eq_take) - min(ex_eq, eq_take));
        const long long p1 = p0 + ngt + taken_eq;
        cluster.sync();  // every selected token of the lane is now visible (cluster-scope acq/rel)
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
                rl[ridx] = (int32_t)p;  // first position; turned into a length below
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
    cluster.sync();  // keep this CTA's shared memory alive until all DSMEM reads are done
}

}  // namespace kvt

using namespace kvt;

constexpr int SEL_SLICE_CAP = 20480;  // 160 KB of staged keys per CTA

extern "C" int kvt_topk_select_runs(const double* cand_score, const int32_t* cand_tok, const int32_t* n_cand,
                         int64_t cand_stride, int64_t n_lanes, int64_t k, int32_t* sel_tok, double* sel_score,
                         int64_t sel_stride, int32_t* n_sel, int32_t* run_start, int32_t* run_len, int64_t run_stride,
                         int32_t* n_runs, void* stream) {
    if (!cand_score || !cand_tok || !n_cand || !sel_tok || !sel_score || !n_sel || n_lanes < 0) return KVT_ERR_ARG;
    if (k < 0) return KVT_ERR_K;
    if (n_lanes == 0) return KVT_OK;
    if (n_lanes > 65535) return KVT_ERR_ARG;
    // cluster size from the largest possible candidate count (cand_stride bounds n_cand)
    int CL = (int)kvt::imin(SEL_MAX_CLUSTER, kvt::imax(1, (cand_stride + 4095) / 4096));
    const int64_t slice = (cand_stride + CL - 1) / CL;
    const int cap = (int)kvt::imin(slice, SEL_SLICE_CAP);
    const size_t smem = (size_t)cap * sizeof(uint64_t);
    KVT_PER_DEVICE(int, g_sel_smem_cap_set);
    if (!g_sel_smem_cap_set) {
        cudaError_t e = cudaFuncSetAttribute(topk_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             SEL_SLICE_CAP * (int)sizeof(uint64_t));
        if (e != cudaSuccess) return kvt_set_cuda_error(e);
        g_sel_smem_cap_set = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, (unsigned)n_lanes, 1);
    cfg.blockDim = dim3(SEL_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, topk_select_kernel, cand_score, cand_tok, n_cand, cand_stride, k, sel_tok,
                                       sel_score, sel_stride, n_sel, cap, run_start, run_len, run_stride, n_runs);
    if (e != cudaSuccess) return kvt_set_cuda_error(e);
    return kvt_check_launch();
}

extern "C" int kvt_topk_select(const double* cand_score, const int32_t* cand_tok, const int32_t* n_cand,
                               int64_t cand_stride, int64_t n_lanes, int64_t k, int32_t* sel_tok, double* sel_score,
                               int64_t sel_stride, int32_t* n_sel, void* stream) {
    return kvt_topk_select_runs(cand_score, cand_tok, n_cand, cand_stride, n_lanes, k, sel_tok, sel_score, sel_stride,
                                n_sel, nullptr, nullptr, 0, nullptr, stream);
}
