// api.cu -- C ABI plumbing: status codes, error text, workspace sizing and the fused
// per-layer pipeline kvt_select_attend (K3 -> plan -> K4 -> K5 -> K6 -> K7), i.e. the body
// of the reference's per-lane loop (engine.py:316-357) for every lane of a layer at once.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>

#include "common.cuh"

static thread_local char g_err[256] = "";

int kvt_set_cuda_error(cudaError_t e) {
    snprintf(g_err, sizeof g_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return KVT_ERR_CUDA;
}

int kvt_set_error_text(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg ? msg : "error");
    return KVT_ERR_CUDA;
}

int kvt_check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return kvt_set_cuda_error(e);
    return KVT_OK;
}

extern "C" int kvt_version(void) { return 100; }  // 0.1.0

extern "C" const char* kvt_status_string(int s) {
    switch (s) {
        case KVT_OK: return "ok";
        case KVT_ERR_SHAPE: return "shape mismatch";
        case KVT_ERR_K: return "k out of range";
        case KVT_ERR_COLD: return "cold chunk but no store was given";
        case KVT_ERR_OOM: return "workspace too small";
        case KVT_ERR_CUDA: return "CUDA error";
        case KVT_ERR_DTYPE: return "unsupported dtype";
        case KVT_ERR_ARG: return "invalid argument";
        default: return "unknown status";
    }
}

extern "C" const char* kvt_last_error(void) { return g_err; }

namespace {

constexpr int ITEM_TOKENS = 64;
constexpr int MAX_SPLITS = 64;

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carve {
    char* p;
    size_t used = 0;
    explicit Carve(void* base) : p((char*)base) {}
    template <typename T> T* take(size_t count) {
        T* r = p ? (T*)(p + used) : nullptr;
        used += align_up(count * sizeof(T));
        return r;
    }
};

struct LayerWs {
    double *U, *L, *A, *err;
    int32_t *items, *n_items, *n_cand;
    double* cand_score;
    float* cs32;
    int32_t* cand_tok;
    char* attn_part;
    unsigned char* qprep;
    size_t bytes;
};

LayerWs carve(void* base, int64_t n_lanes, int64_t n, int64_t max_leaves, int d) {
    Carve c(base);
    LayerWs w;
    const int64_t item_cap = (n + ITEM_TOKENS - 1) / ITEM_TOKENS + max_leaves;
    // the attention region goes first: its merge tickets must stay zero between calls, and
    // its offset must not depend on max_leaves, which changes with the layer's chunk size
    w.attn_part = c.take<char>(kvt_attn_workspace_bytes(n_lanes, d, MAX_SPLITS));  // tickets + lse + partials
    w.U = c.take<double>((size_t)(n_lanes * max_leaves));
    w.L = c.take<double>((size_t)(n_lanes * max_leaves));
    w.A = c.take<double>((size_t)(n_lanes * max_leaves));
    w.err = c.take<double>((size_t)(n_lanes * 4));
    w.items = c.take<int32_t>((size_t)(n_lanes * item_cap * 3));
    w.n_items = c.take<int32_t>((size_t)n_lanes);
    w.n_cand = c.take<int32_t>((size_t)n_lanes);
    w.cand_score = c.take<double>((size_t)(n_lanes * n));
    w.cand_tok = c.take<int32_t>((size_t)(n_lanes * n));
    w.cs32 = c.take<float>((size_t)(n_lanes * n));
    w.qprep = c.take<unsigned char>(kvt_i4_qprep_bytes(n_lanes, d));              // INT4 query digits
    w.bytes = c.used;
    return w;
}

// A per-thread side stream + fork/join events: the INT4 query-digit prep (depends on q only)
// runs concurrently with bounds and plan; inside CUDA-graph capture it becomes a parallel branch.
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    bool ok = false;
    SideStream() {
        ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
        if (!ok) cudaGetLastError();
    }
};
SideStream& side_stream() {  // one per thread and device (streams belong to a device)
    static thread_local SideStream* ss[kvt::kMaxDevices] = {};
    const int dev = kvt::current_device();
    if (!ss[dev]) ss[dev] = new SideStream();  // lives as long as the thread's CUDA context use
    return *ss[dev];
}

int num_sms() { return kvt::sm_count(); }

// GQA union attention in kvt_select_attend: opt-in with KVT_GQA_UNION=1.  The per-query-lane
// ring kernel is the default: at config 4 it measures 20.46 ms per step against 21.06 with the
// union (whose smaller V read does not pay for its window plan pass; DESIGN.md section 0 +B).
bool gqa_union_on() {
    const char* e = getenv("KVT_GQA_UNION");
    return e && e[0] == '1';
}

}  // namespace

extern "C" size_t kvt_layer_workspace_bytes(int64_t n_lanes, int64_t n, int64_t max_leaves, int d) {
    return carve(nullptr, n_lanes, n, max_leaves, d).bytes;
}

int& kv_group_tls() {
    static thread_local int g = 1;
    return g;
}

float*& sel_hint_tls() {
    static thread_local float* h = nullptr;
    return h;
}

int& cand_group_tls() {
    static thread_local int g = 1;
    return g;
}

extern "C" int kvt_set_cand_group(int g) {
    const int old = cand_group_tls();
    cand_group_tls() = g > 1 ? g : 1;
    return old;
}

extern "C" int kvt_set_kv_group(int kv_group) {
    const int old = kv_group_tls();
    kv_group_tls() = kv_group > 1 ? kv_group : 1;
    return old;
}

extern "C" int kvt_select_attend(const kvt_layer_args* a, void* ws, size_t ws_bytes, void* stream) {
    if (!a || !ws) return KVT_ERR_ARG;
    const int kvg = a->kv_group > 1 ? a->kv_group : 1;
    if (kvg > 1 && (a->n_lanes % kvg || !a->abs_mag || a->abs_dtype != KVT_BF16 || a->q_dtype != KVT_F32 ||
                    a->leaf_start || a->exact_scores || !kvt_fast_ok(a->key_dtype, a->d)))
        return KVT_ERR_ARG;  // GQA sharing runs on the decode path's kernels only
    KvGroupScope group_scope(kvg);
    SelHintScope hint_scope(a->sel_hint);
    if (a->k < 0 || a->k > a->n) return KVT_ERR_K;
    if (a->n_lanes <= 0 || a->n <= 0) return a->n_lanes == 0 ? KVT_OK : KVT_ERR_ARG;
    if (!a->leaf_start && a->C < 1) return KVT_ERR_ARG;
    const int64_t max_leaves = a->leaf_start ? a->leaf_stride : (a->n + a->C - 1) / a->C;
    LayerWs w = carve(ws, a->n_lanes, a->n, max_leaves, a->d);
    if (w.bytes > ws_bytes) return KVT_ERR_OOM;
    const int64_t item_cap = (a->n + ITEM_TOKENS - 1) / ITEM_TOKENS + max_leaves;
    int rc;
    // fast path: f32 estimates + exact band re-scoring (any key dtype but f64, d = 128/256)
    const bool fast = kvt_fast_ok(a->key_dtype, a->d) && !a->exact_scores;
    const bool fast_bounds = fast && a->abs_mag && a->abs_dtype == KVT_BF16 && a->q_dtype == KVT_F32 &&
                             !a->leaf_start && (a->d == 128 || a->d == 256);
    // INT4 fast path: query digits on the side stream, joined before the scoring launch
    const bool i4_fast = fast && a->key_dtype == KVT_I4;
    SideStream& ss = side_stream();
    const bool forked = i4_fast && ss.ok;
    if (forked) {
        cudaEventRecord(ss.fork, (cudaStream_t)stream);
        cudaStreamWaitEvent(ss.s, ss.fork, 0);
        rc = kvt_i4_qprep(a->q, a->q_dtype, a->n_lanes, a->d, w.qprep, ss.s);
        if (rc) return rc;
        cudaEventRecord(ss.join, ss.s);
    }
    if (fast_bounds)  // sound f32 directed-rounding bounds (bounds_fast.cu)
        rc = kvt_chunk_bounds_fast((const float*)a->q, a->n_lanes, a->d, a->n, a->C, a->amax, a->amin,
                                   a->abs_lane_stride, a->abs_mag, w.U, w.L, w.A, max_leaves, stream);
    else
        rc = kvt_chunk_bounds(a->q, a->q_dtype, a->n_lanes, a->d, a->n, a->C, a->leaf_start, a->n_leaves,
                              a->leaf_stride, a->amax, a->amin, a->abs_dtype, a->abs_lane_stride, w.U, w.L,
                              fast ? w.A : nullptr, max_leaves, 0, stream);
    if (rc) return rc;
    // GQA with INT4 keys: one candidate list per KV lane (union over its query lanes), scored
    // once for the whole group (score_i4mma QG > 1); selectors read the shared token-id row
    const int ugrp = (kvg > 1 && i4_fast) ? kvg : 1;
    CandGroupScope cand_scope(ugrp);
    rc = kvt_select_plan_group(a->n_lanes, a->n, a->C, a->leaf_start, a->n_leaves, a->leaf_stride, w.U, w.L,
                               max_leaves, a->k, w.items, item_cap, w.n_items, w.n_cand, nullptr, a->evals,
                               fast ? w.A : nullptr, fast ? w.err : nullptr, a->d, ugrp, stream);
    if (rc) return rc;
    if (fast) {
        if (a->key_dtype == KVT_I4)  // exact int32 inner products on the tensor cores + per-lane bound
        {
            if (forked) cudaStreamWaitEvent((cudaStream_t)stream, ss.join, 0);
            rc = kvt_cand_score_i4mma(forked ? nullptr : a->q, a->q_dtype, a->keys, a->n_lanes, a->lane_stride, a->d,
                                      w.items, item_cap,
                                      w.n_items, w.cs32, w.cand_tok, a->n, w.err, w.qprep, stream);
        } else
            rc = kvt_cand_score_f32(a->q, a->q_dtype, a->keys, a->key_dtype, a->n_lanes, a->lane_stride, a->d, w.items,
                                    item_cap, w.n_items, w.cs32, w.cand_tok, a->n, stream);
        if (rc) return rc;
        rc = kvt_topk_select_band(w.cs32, w.cand_tok, w.n_cand, a->n, w.err, a->n_lanes, a->k, a->q, a->q_dtype,
                                  a->keys, a->key_dtype, a->lane_stride, a->d, w.cand_score, a->sel_tok,
                                  a->sel_score, a->k, a->n_sel, a->run_start, a->run_len, a->k, a->n_runs, stream);
        if (rc) return rc;
    } else {

        int blocks = a->score_blocks;
        if (blocks <= 0) {
            const int64_t target = (int64_t)num_sms() * 8;  // 8 CTAs of 256 threads per SM
            const int64_t per_lane = (target + a->n_lanes - 1) / a->n_lanes;
            const int64_t need = (item_cap + 7) / 8;
            blocks = (int)kvt::imax(1, kvt::imin(per_lane, need));
        }
        rc = kvt_cand_score(a->q, a->q_dtype, a->keys, a->key_dtype, a->n_lanes, a->lane_stride, a->d, w.items, item_cap,
                            w.n_items, w.cand_score, w.cand_tok, a->n, blocks, stream);
        if (rc) return rc;
        rc = kvt_topk_select_runs(w.cand_score, w.cand_tok, w.n_cand, a->n, a->n_lanes, a->k, a->sel_tok, a->sel_score,
                                  a->k, a->n_sel, a->run_start, a->run_len, a->k, a->n_runs, stream);  // K5 + fused K6
        if (rc) return rc;

    }
    if (a->out && a->values && kvg > 1 && a->v_dtype == KVT_I4 && a->attn_splits <= 0 && gqa_union_on()) {
        // GQA: one pass over the group's union, P.V on the tensor cores (attn_gqa.cu); the
        // candidate-score region (only used by the exact fallback, done by now) is its scratch
        const size_t sb = (size_t)a->n_lanes * (size_t)a->n * sizeof(double);
        rc = kvt_sparse_decode_attn_gqa(a->values, a->n_lanes, a->lane_stride, a->d, kvg, a->n, a->sel_tok,
                                        a->sel_score, a->n_sel, a->k, 1.0 / sqrt((double)a->d), w.attn_part,
                                        w.cand_score, sb, a->out, nullptr, stream);
        if (rc != KVT_ERR_ARG) return rc;  // else: a shape the union kernel does not cover
    }
    if (a->out && a->values) {
        int splits = a->attn_splits;  // 0 = auto: wave-aware choice in kvt_sparse_decode_attn
        if (splits > MAX_SPLITS) splits = MAX_SPLITS;
        rc = kvt_sparse_decode_attn(a->values, a->v_dtype, a->n_lanes, a->lane_stride, a->d, a->sel_tok, a->sel_score,
                                    a->n_sel, a->k, 1.0 / sqrt((double)a->d), splits, w.attn_part, a->out, nullptr,
                                    stream);
        if (rc) return rc;
    }
    return KVT_OK;
}
