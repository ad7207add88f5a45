// tier.cu -- the GPU side of the tiered KV store (north-star item 5).
//
// The reference moves whole placement records between tiers with fetch_chunk / promote_hot /
// ensure_hot and evicts the least recently touched record first, ordered by
// (last_touch, start, layer, head) (tiered_store.py:224-372), driven per lane from
// engine.py:342-343 (store.touch(selected); store.ensure_hot(_token_runs(selected))).
// Here the tiers are real memory: the HOT tier is a pool of record slots in HBM, the WARM
// tier the pinned host copy of every record, read by the GPU over the host link (mapped,
// zero-copy).  One call per (step, layer) does, stream-ordered and without a host round trip:
//   touch    the records the layer's selected runs overlap: hits get stamp = step, misses
//            are claimed once (table entry -1 -> -2) and appended to the miss list;
//   prep     M = misses, free slots F, evictions E = max(0, M - F);
//   victims  the E least recently touched hot records, exactly the reference's order: key =
//            (stamp, record id) with id = (start record, layer, lane) -- a 3-pass radix select
//            (13-bit digits) over the slot keys, records touched in this step excluded;
//   assign   victims go hot -> warm (table entry -1), misses get slots (table, owner, stamp);
//            the row's ledger counters (warm_to_hot, hot_to_warm, fetch_ops) are summed;
//   fetch    one warp per miss copies the record host -> HBM slot: INT4 records as stored, or
//            (for the theta-split's raw share) bf16 rows quantised on the fly with the K8
//            codec, so the slot's codes are the same either way.
// K7 then reads V through the slot table (kvt_sparse_decode_attn_paged).
// Stamps older than 4095 steps compare as equally old (ties by record id).
#include <cuda_fp16.h>

#include "common.cuh"
#include "quant_codec.cuh"

namespace kvt {
namespace {

constexpr int TB = 256;
constexpr int DIG = 13, NBIN = 1 << DIG;
constexpr int AGE_BITS = 12;

struct TierCtl {            // device control block (kvt_tier_ctl_bytes)
    int32_t miss_count;     // touch appends here; prep moves it to m
    int32_t m, nfree, evict;
    int32_t need;           // radix select: evictions still to place at the current digit
    int32_t n_victims;
    int32_t pad[2];
    unsigned long long prefix, mask;
};

// Eviction key of a hot record: (stamp, start record, layer, lane) -- the reference's
// (last_touch, start, layer, head) -- packed as age (12 bits, 0 = oldest) | rec * n_lk + lk,
// where the owner id is lk * n_rec + rec and lk = layer * kv_lanes + lane.
__device__ __forceinline__ unsigned long long slot_key(int32_t stamp, long long id, int step, long long n_rec,
                                                       long long n_lk) {
    const int age_base = step - ((1 << AGE_BITS) - 1);
    const int rel = stamp < age_base ? 0 : stamp - age_base;
    const long long rec = id % n_rec, lk = id / n_rec;
    return ((unsigned long long)rel << 26) | (unsigned long long)(rec * n_lk + lk);
}

__global__ void tier_touch_kernel(const int32_t* __restrict__ run_start, const int32_t* __restrict__ run_len,
                                  const int32_t* __restrict__ n_runs, int64_t run_stride, int kvg, int crec,
                                  int32_t* table, int64_t table_stride, int64_t table_base, int32_t* stamp,
                                  const int32_t* __restrict__ step_p, int64_t* miss, int64_t miss_cap, TierCtl* ctl) {
    const int step = *step_p;
    const int64_t li = blockIdx.x;
    const int64_t kvl = li / kvg;
    const int nr = n_runs[li];
    const int32_t* rs = run_start + li * run_stride;
    const int32_t* rl = run_len + li * run_stride;
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
        const int s = rs[r], e = s + rl[r];
        for (int rec = s / crec; rec <= (e - 1) / crec; ++rec) {
            int32_t* t = table + kvl * table_stride + rec;
            const int32_t v = *reinterpret_cast<volatile int32_t*>(t);
            if (v >= 0) {
                stamp[v] = step;
            } else if (v == -1 && atomicCAS(t, -1, -2) == -1) {
                const int i = atomicAdd(&ctl->miss_count, 1);
                if (i < miss_cap) miss[i] = table_base + kvl * table_stride + rec;
            }
        }
    }
}

__global__ void tier_prep_kernel(TierCtl* ctl, const int32_t* free_top, int64_t miss_cap, unsigned int* hist) {
    for (int i = threadIdx.x; i < NBIN; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
        const int m = (int)min((int64_t)ctl->miss_count, miss_cap);
        ctl->miss_count = 0;
        ctl->m = m;
        ctl->nfree = *free_top;
        ctl->evict = max(0, m - ctl->nfree);
        ctl->need = ctl->evict;
        ctl->n_victims = 0;
        ctl->prefix = 0;
        ctl->mask = 0;
    }
}

// eligible = occupied and not touched in this step
__global__ void tier_hist_kernel(const int64_t* __restrict__ owner, const int32_t* __restrict__ stamp,
                                 int64_t n_slots, const int32_t* __restrict__ step_p, int64_t n_rec, int64_t n_lk,
                                 int shift, const TierCtl* ctl, unsigned int* hist) {
    if (ctl->need <= 0) return;
    const int step = *step_p;
    const unsigned long long pf = ctl->prefix, mk = ctl->mask;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += (int64_t)gridDim.x * blockDim.x) {
        const long long id = owner[i];
        const int32_t st = stamp[i];
        if (id < 0 || st >= step) continue;
        const unsigned long long key = slot_key(st, id, step, n_rec, n_lk);
        if ((key & mk) != pf) continue;
        atomicAdd(&hist[(key >> shift) & (NBIN - 1)], 1u);
    }
}

// one CTA: the digit (ascending = least recently used first) where the running count reaches
// `need`; narrows prefix/mask, leaves need = the count still to take inside that digit
__global__ void tier_find_kernel(TierCtl* ctl, unsigned int* hist, int shift) {
    __shared__ long long sh[33];
    __shared__ int s_digit;
    __shared__ long long s_before;
    const int tid = threadIdx.x;
    const int need = ctl->need;
    if (need <= 0) return;  // block-uniform
    constexpr int PER = NBIN / 1024;
    long long loc = 0;
    for (int j = 0; j < PER; ++j) loc += hist[tid * PER + j];
    long long tot;
    const long long ex = block_excl_scan<long long>(loc, sh, tot);
    if (tid == 0) { s_digit = -1; s_before = 0; }
    __syncthreads();
    if (ex < need && need <= ex + loc) {
        long long run = ex;
        for (int j = 0; j < PER; ++j) {
            const long long c = hist[tid * PER + j];
            if (run + c >= need) { s_digit = tid * PER + j; s_before = run; break; }
            run += c;
        }
    }
    __syncthreads();
    for (int j = 0; j < PER; ++j) hist[tid * PER + j] = 0;  // ready for the next pass
    if (tid == 0) {
        if (s_digit < 0) {  // fewer eligible records than evictions: the step's working set
            ctl->need = -1;  // does not fit (CapacityError on the host)
        } else {
            ctl->prefix |= (unsigned long long)s_digit << shift;
            ctl->mask |= (unsigned long long)(NBIN - 1) << shift;
            ctl->need = (int)(need - s_before);
        }
    }
}

// victims = eligible slots whose key <= the boundary key (keys are unique: exactly E)
__global__ void tier_gather_kernel(const int64_t* __restrict__ owner, const int32_t* __restrict__ stamp,
                                   int64_t n_slots, const int32_t* __restrict__ step_p, int64_t n_rec, int64_t n_lk,
                                   TierCtl* ctl, int32_t* victims) {
    if (ctl->evict <= 0 || ctl->need < 0) return;
    const int step = *step_p;
    const unsigned long long bound = ctl->prefix;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += (int64_t)gridDim.x * blockDim.x) {
        const long long id = owner[i];
        const int32_t st = stamp[i];
        if (id < 0 || st >= step) continue;
        if (slot_key(st, id, step, n_rec, n_lk) <= bound) victims[atomicAdd(&ctl->n_victims, 1)] = (int32_t)i;
    }
}

// j < M: slot = a free slot (stack top first) or victim j - F
__global__ void tier_assign_kernel(const int64_t* __restrict__ miss, TierCtl* ctl, int32_t* free_stack, int32_t* free_top,
                                   const int32_t* __restrict__ victims, int32_t* table, int64_t* owner, int32_t* stamp,
                                   int32_t* slot_of_miss, const int32_t* __restrict__ step_p, long long ledger_rec_bytes,
                                   unsigned long long* ledger_row) {
    const int m = ctl->m, nf = ctl->nfree;
    const int step = *step_p;
    if (ctl->need < 0) {  // (grid-uniform) capacity error: flagged in the row
        if (blockIdx.x == 0 && threadIdx.x == 0) ledger_row[3] = ~0ull;
        return;
    }
    unsigned long long w2h = 0, h2w = 0, ops = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        int32_t slot;
        if (j < nf) {
            slot = free_stack[nf - 1 - j];
        } else {
            slot = victims[j - nf];
            table[owner[slot]] = -1;  // hot -> warm: the host copy is already there (write-through)
            h2w += (unsigned long long)ledger_rec_bytes;
        }
        const long long id = miss[j];
        table[id] = slot;
        owner[slot] = id;
        stamp[slot] = step;
        slot_of_miss[j] = slot;
        w2h += (unsigned long long)ledger_rec_bytes;
        ops += 1;
    }
    // ledger row: warp sums, one atomic per warp
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        w2h += __shfl_xor_sync(KVT_FULL, w2h, o);
        h2w += __shfl_xor_sync(KVT_FULL, h2w, o);
        ops += __shfl_xor_sync(KVT_FULL, ops, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (w2h) atomicAdd(&ledger_row[0], w2h);
        if (h2w) atomicAdd(&ledger_row[1], h2w);
        if (ops) atomicAdd(&ledger_row[2], ops);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *free_top = nf - min(m, nf);
}

__device__ __forceinline__ uint4 ld_host16(const void* p) {  // host-mapped, read once
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// one warp per miss.  id = (layer row base + kv lane * n_rec + rec); the host copies are
// [kv lanes][N][row] per layer, so record rec of lane kvl starts at token rec * crec.
template <int D>
__global__ void __launch_bounds__(TB) tier_fetch_kernel(const int64_t* __restrict__ miss, const int32_t* __restrict__ slot_of_miss,
                                                        const TierCtl* ctl, int64_t table_base, int64_t table_stride,
                                                        int crec, int64_t n_tok, const unsigned char* __restrict__ host_i4,
                                                        const __nv_bfloat16* __restrict__ host_raw, int64_t host_lane_tokens,
                                                        const float* __restrict__ theta_p, unsigned char* __restrict__ pool) {
    constexpr int RB = D / 2 + D / 8;
    const int m = ctl->m;
    if (ctl->need < 0) return;
    const float theta = theta_p ? fminf(fmaxf(*theta_p, 0.f), 1.f) : 1.f;
    const int n_comp = host_raw ? (int)ceilf(theta * (float)m - 1e-6f) : m;
    const int lane = threadIdx.x & 31;
    for (int j = blockIdx.x * (TB / 32) + (threadIdx.x >> 5); j < m; j += gridDim.x * (TB / 32)) {
        const long long id = miss[j] - table_base;
        const long long kvl = id / table_stride, rec = id % table_stride;
        const long long t0 = rec * crec;
        const int nt = (int)min((long long)crec, n_tok - t0);
        unsigned char* dst = pool + (size_t)slot_of_miss[j] * crec * RB;
        if (j < n_comp) {  // compressed: the INT4 record bytes as stored
            const unsigned char* src = host_i4 + ((size_t)kvl * host_lane_tokens + t0) * RB;
            const int n16 = nt * RB / 16;
            constexpr int U = 4;
            for (int b = lane; b < n16; b += 32 * U) {
                uint4 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b + 32 * u < n16) x[u] = ld_host16(src + 16 * (size_t)(b + 32 * u));
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b + 32 * u < n16) *reinterpret_cast<uint4*>(dst + 16 * (size_t)(b + 32 * u)) = x[u];
            }
        } else {  // raw bf16 rows over the link, quantised here (same codes as K8)
            const __nv_bfloat16* src = host_raw + ((size_t)kvl * host_lane_tokens + t0) * D;
            constexpr int IPR = D / 8;  // items per row
            for (int base = 0; base < nt * IPR; base += 32) {  // warp-uniform: every lane shuffles
                const int it = base + lane;
                const bool ok = it < nt * IPR;
                const int t = it / IPR, c = it % IPR;
                const uint4 a = ok ? ld_host16(src + (size_t)t * D + 8 * c) : make_uint4(0, 0, 0, 0);
                const uint32_t w[4] = {a.x, a.y, a.z, a.w};
                float f[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    f[2 * i] = __uint_as_float(w[i] << 16);
                    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
                }
                float lo = f[0], hi = f[0];
#pragma unroll
                for (int e = 1; e < 8; ++e) { lo = fminf(lo, f[e]); hi = fmaxf(hi, f[e]); }
                bool big = false;
#pragma unroll
                for (int e = 0; e < 8; ++e) big |= fabsf(f[e]) > 65504.0f;
                __half sh, mh;
                const uint32_t code = __any_sync(KVT_FULL, big) ? quant_item<true>(f, lo, hi, sh, mh)
                                                                : quant_item<false>(f, lo, hi, sh, mh);
                if (!ok) continue;
                unsigned char* row = dst + (size_t)t * RB;
                *reinterpret_cast<uint32_t*>(row + 4 * c) = code;
                if ((c & 3) == 0) {
                    __half2 p = __halves2half2(sh, mh);
                    *reinterpret_cast<__half2*>(row + D / 2 + 4 * (c >> 2)) = p;
                }
            }
        }
    }
}

inline int grid_for(int64_t n) { return (int)kvt::imax(1, kvt::imin((int64_t)kvt::sm_count() * 4, (n + TB - 1) / TB)); }

}  // namespace
}  // namespace kvt

using namespace kvt;

extern "C" size_t kvt_tier_ctl_bytes(void) { return sizeof(TierCtl) + NBIN * sizeof(unsigned int); }

extern "C" int kvt_tier_layer(const kvt_tier_args* a, void* stream) {
    if (!a || !a->table || !a->stamp || !a->owner || !a->free_stack || !a->free_top || !a->pool || !a->ctl ||
        !a->miss || !a->slot_of_miss || !a->victims || !a->host_i4 || !a->run_start || !a->run_len || !a->n_runs ||
        !a->ledger_row)
        return KVT_ERR_ARG;
    if (a->d != 128 && a->d != 256) return KVT_ERR_SHAPE;
    if (a->crec < 1 || a->n_lanes < 0 || a->kv_group < 1 || a->n_lanes % a->kv_group) return KVT_ERR_ARG;
    if (a->table_stride < 1 || a->n_lk < 1 || a->table_stride * a->n_lk > (1LL << 26) || a->n_slots < 0 ||
        a->n_slots > 0x7fffffffLL)
        return KVT_ERR_ARG;  // record ids must fit the 26-bit key field
    if (a->n_lanes == 0) return KVT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    TierCtl* ctl = (TierCtl*)a->ctl;
    unsigned int* hist = (unsigned int*)((char*)a->ctl + sizeof(TierCtl));
    int32_t* table_l = a->table + a->table_base;
    tier_touch_kernel<<<(unsigned)a->n_lanes, TB, 0, st>>>(a->run_start, a->run_len, a->n_runs, a->run_stride,
                                                           a->kv_group, a->crec, table_l, a->table_stride, a->table_base,
                                                           a->stamp, a->step, a->miss, a->miss_cap, ctl);
    tier_prep_kernel<<<1, 1024, 0, st>>>(ctl, a->free_top, a->miss_cap, hist);
    const int g = grid_for(a->n_slots);
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = 2 * DIG - DIG * pass;  // 26, 13, 0: key bits [26, 39), [13, 26), [0, 13)
        tier_hist_kernel<<<g, TB, 0, st>>>(a->owner, a->stamp, a->n_slots, a->step, a->table_stride, a->n_lk, shift,
                                           ctl, hist);
        tier_find_kernel<<<1, 1024, 0, st>>>(ctl, hist, shift);
    }
    tier_gather_kernel<<<g, TB, 0, st>>>(a->owner, a->stamp, a->n_slots, a->step, a->table_stride, a->n_lk, ctl,
                                         a->victims);
    const int ga = grid_for(a->miss_cap);
    tier_assign_kernel<<<ga, TB, 0, st>>>(a->miss, ctl, a->free_stack, a->free_top, a->victims, a->table, a->owner,
                                          a->stamp, a->slot_of_miss, a->step, a->ledger_rec_bytes,
                                          (unsigned long long*)a->ledger_row);
    const int gf = (int)kvt::imax(1, kvt::imin((int64_t)kvt::sm_count() * 8, (a->miss_cap + 7) / 8));
    if (a->d == 128)
        tier_fetch_kernel<128><<<gf, TB, 0, st>>>(a->miss, a->slot_of_miss, ctl, a->table_base, a->table_stride,
                                                  a->crec, a->n_tok, (const unsigned char*)a->host_i4,
                                                  (const __nv_bfloat16*)a->host_raw, a->host_lane_tokens, a->theta,
                                                  (unsigned char*)a->pool);
    else
        tier_fetch_kernel<256><<<gf, TB, 0, st>>>(a->miss, a->slot_of_miss, ctl, a->table_base, a->table_stride,
                                                  a->crec, a->n_tok, (const unsigned char*)a->host_i4,
                                                  (const __nv_bfloat16*)a->host_raw, a->host_lane_tokens, a->theta,
                                                  (unsigned char*)a->pool);
    return kvt_check_launch();
}

// State of the last kvt_tier_layer call: out4 = [m misses, evictions, need (< 0: the step's
// working set did not fit), victims found].  Synchronises the stream (tests / diagnostics).
extern "C" int kvt_tier_read_ctl(const void* ctl_dev, long long* out4, void* stream) {
    if (!ctl_dev || !out4) return KVT_ERR_ARG;
    TierCtl h;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(&h, ctl_dev, sizeof(TierCtl), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return kvt_set_cuda_error(e);
    out4[0] = h.m;
    out4[1] = h.evict;
    out4[2] = h.need;
    out4[3] = h.n_victims;
    return KVT_OK;
}
