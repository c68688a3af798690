// msd_api.cu -- the C ABI of libmsd (declared and documented in include/msd.h):
// argument validation, workspace carving and kernel launches.  No arithmetic of
// the method lives here.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "msd_common.cuh"
#include "msd_internal.h"

using namespace msd;

namespace msd {
DebugKnobs g_knobs;
}

namespace {

thread_local std::string g_err;

msd_status fail(msd_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

msd_status cuda_fail(cudaError_t e, const char* where) {
    return fail(MSD_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

msd_status check_arch() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    static int cached[64];
    static std::once_flag once[64];
    if (dev < 0 || dev >= 64) return fail(MSD_E_ARCH, "device index %d", dev);
    std::call_once(once[dev], [&]() {
        int major = 0, minor = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        cached[dev] = major * 10 + minor;
    });
    if (cached[dev] != 100)
        return fail(MSD_E_ARCH, "libmsd is built for sm_100a (B200); device %d is sm_%d", dev,
                    cached[dev]);
    return MSD_OK;
}


// One-time per-device setup (the bf16 exp table of the tail's exact draws), under call_once:
// on a private stream with a wait on that stream only, so it must not run while another stream
// of the process is being captured into a CUDA graph -- call msd_init first in that case.
msd_status device_init() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    static std::once_flag once[64];
    static cudaError_t res[64];
    if (dev < 0 || dev >= 64) return fail(MSD_E_ARCH, "device index %d", dev);
    std::call_once(once[dev], [&]() {
        const double* t = nullptr;
        res[dev] = exp_table(&t, 1);
    });
    if (res[dev] != cudaSuccess) return cuda_fail(res[dev], "msd_init");
    return MSD_OK;
}

// Workspace binding: the exchange records of a workspace are laid out for one (L, B, K, V);
// a workspace seen with another shape (or for the first time) gets its record region zeroed
// on the call's stream before use (msd.h workspace contract).
std::mutex g_ws_mu;
std::vector<std::pair<const void*, uint64_t>> g_ws_shape;
bool ws_shape_changed(const void* ws, uint64_t key) {
    std::lock_guard<std::mutex> g(g_ws_mu);
    for (auto& e : g_ws_shape)
        if (e.first == ws) {
            const bool ch = e.second != key;
            e.second = key;
            return ch;
        }
    if (g_ws_shape.size() >= 256) g_ws_shape.erase(g_ws_shape.begin());
    g_ws_shape.emplace_back(ws, key);
    return true;
}

unsigned long long* g_trace = nullptr;   // debug trace buffer (msd_debug_set_trace)
size_t g_trace_items = 0;

// ----------------------------------------------------------------- profiling
struct Prof {
    std::mutex mu;
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
    int32_t total_launches = 0;
} g_prof;

std::pair<cudaEvent_t, cudaEvent_t> prof_pair() {
    std::pair<cudaEvent_t, cudaEvent_t> p;
    if (!g_prof.pool.empty()) {
        p = g_prof.pool.back();
        g_prof.pool.pop_back();
    } else {
        cudaEventCreate(&p.first);
        cudaEventCreate(&p.second);
    }
    return p;
}

struct Engine {
    LevelDesc lv;
    int32_t L, B, K;
    int64_t V;
    int32_t bf16;
    const int32_t* cand0;
    const int32_t* m0;
    const float* u_acc;
    const float* u_emit;
    int64_t ua_l, ua_b, ue_l, ue_b;
    int32_t greedy, ibonus, fbonus, draft_fed;
    int32_t *n_acc, *m_cand, *out_tok, *out_len, *rollback;
    int32_t out_ld;
    float *pos_dtv, *pos_kl;
    msd_pair_stats* stats;
    uint32_t* flags;
    void* ws;
    size_t ws_bytes;
    cudaStream_t stream;
    float inv_temp;     // logits processor: 1 / temperature (1 = none)
    const double* lse;  // producer-supplied row normalisers [L][B][K] (msd_chain_verify_lse) or NULL
};

msd_status validate_levels(const msd_logits* lv, int32_t L, int32_t K, int64_t V, int32_t ibonus,
                           int32_t extra_rows_needed, int32_t* bf16) {
    const int32_t dt = lv[0].dtype;
    if (dt != MSD_F32 && dt != MSD_BF16) return fail(MSD_E_DTYPE, "unknown dtype %d", dt);
    const int64_t es = dt == MSD_BF16 ? 2 : 4;
    for (int l = 0; l < L; ++l) {
        if (lv[l].dtype != dt) return fail(MSD_E_DTYPE, "level %d dtype differs from level 0", l);
        if (!lv[l].ptr) return fail(MSD_E_ARG, "level %d ptr is NULL", l);
        if (lv[l].ld < V) return fail(MSD_E_ARG, "level %d ld=%lld < V=%lld", l, (long long)lv[l].ld, (long long)V);
        int32_t need = l == 0 ? K : (extra_rows_needed >= 0 ? K + extra_rows_needed : (ibonus ? K + l : K + 1));
        if (lv[l].rows < need) return fail(MSD_E_ARG, "level %d has %d rows, needs >= %d", l, lv[l].rows, need);
        if (lv[l].batch_stride < (int64_t)lv[l].rows * lv[l].ld)
            return fail(MSD_E_ARG, "level %d batch_stride < rows*ld", l);
        if (((uintptr_t)lv[l].ptr) % 16 || (lv[l].ld * es) % 16 || (lv[l].batch_stride * es) % 16)
            return fail(MSD_E_ALIGN, "level %d rows are not 16-byte aligned (ptr, ld*elem, batch_stride*elem)", l);
    }
    *bf16 = dt == MSD_BF16;
    return MSD_OK;
}

msd_status run_engine(const Engine& E) {
    if (E.B == 0) return MSD_OK;
    const WsLayout w = ws_layout(E.L, E.B, E.K, E.V);
    if (!E.ws || E.ws_bytes < w.total)
        return fail(MSD_E_WORKSPACE, "workspace %zu bytes < required %zu", E.ws_bytes, w.total);
    if (((uintptr_t)E.ws) % 256) return fail(MSD_E_WORKSPACE, "workspace must be 256-byte aligned");
    char* ws = reinterpret_cast<char*>(E.ws);
    {
        const uint64_t key = ((uint64_t)E.L << 60) ^ ((uint64_t)E.B << 40) ^ ((uint64_t)E.K << 32) ^ (uint64_t)E.V;
        if (ws_shape_changed(E.ws, key)) {
            cudaError_t me = cudaMemsetAsync(ws + w.partms, 0, w.rowstat - w.partms, E.stream);
            if (me != cudaSuccess) return cuda_fail(me, "workspace reset");
        }
    }

    CoreParams cp;
    memset(&cp, 0, sizeof(cp));
    cp.lv = E.lv;
    cp.L = E.L; cp.B = E.B; cp.K = E.K; cp.V = E.V;
    cp.C = w.C; cp.U = w.U; cp.VSe = slice_geometry(E.V).VSe;
    cp.kinv = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)E.K - 1) / (uint64_t)E.K);
    if (w.U >= (1 << 24)) return fail(MSD_E_ARG, "B*K = %d units exceeds 2^24", w.U);
    cp.n_items = (int64_t)w.U * w.C;
    cp.partials = reinterpret_cast<Partial*>(ws + w.partials);
    cp.partms = reinterpret_cast<float2*>(ws + w.partms);
    cp.rowstat = reinterpret_cast<RowStat*>(ws + w.rowstat);
    cp.kl = reinterpret_cast<double*>(ws + w.kl);
    cp.resid = reinterpret_cast<double*>(ws + w.resid);
    cp.cnt = reinterpret_cast<uint32_t*>(ws + w.cnt);
    cp.ready = reinterpret_cast<uint32_t*>(ws + w.ready);
    cp.flags = E.flags;
    cp.err = reinterpret_cast<uint32_t*>(ws + w.hdr);
    cp.board = reinterpret_cast<JobBoard*>(ws + w.board);
    cp.trace = (g_trace && g_trace_items >= (size_t)cp.n_items) ? g_trace : nullptr;
    cp.dbg = g_knobs.core_dbg;
    cp.inv_temp = E.inv_temp;
    cp.lse = E.lse;

    TailParams tp;
    memset(&tp, 0, sizeof(tp));
    tp.lv = E.lv;
    tp.L = E.L; tp.B = E.B; tp.K = E.K; tp.C = w.C; tp.V = E.V; tp.VSe = cp.VSe;
    tp.cand0 = E.cand0; tp.m0 = E.m0;
    tp.u_acc = E.u_acc; tp.u_emit = E.u_emit;
    tp.ua_l = E.ua_l; tp.ua_b = E.ua_b; tp.ue_l = E.ue_l; tp.ue_b = E.ue_b;
    tp.greedy = E.greedy; tp.ibonus = E.ibonus; tp.fbonus = E.fbonus; tp.draft_fed = E.draft_fed;
    tp.n_acc = E.n_acc; tp.m_cand = E.m_cand; tp.out_tok = E.out_tok; tp.out_ld = E.out_ld;
    tp.out_len = E.out_len; tp.rollback = E.rollback;
    tp.pos_dtv = E.pos_dtv; tp.pos_kl = E.pos_kl; tp.stats = E.stats; tp.flags = E.flags;
    tp.partials = cp.partials; tp.partms = cp.partms; tp.resid = cp.resid;
    tp.cnt = cp.cnt;
    tp.board = cp.board;
    tp.inv_temp = E.inv_temp;
    tp.z_safe = g_knobs.z_safe;                  // exact draws below this residual mass (R4)
    tp.exact_all = g_knobs.exact_draws;
    {
        msd_status is = device_init();
        if (is != MSD_OK) return is;
        cudaError_t te = exp_table(&tp.exptab, 0);
        if (te != cudaSuccess) return cuda_fail(te, "exp table");
    }

    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    // under stream capture (a CUDA graph) the events become external event-record nodes, which
    // record on every replay (a plain record would only add a capture dependency)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(E.stream, &cap);
    const unsigned rec_flags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    {
        std::lock_guard<std::mutex> g(g_prof.mu);
        if (g_prof.on) {
            ev = prof_pair();
            cudaEventRecordWithFlags(ev.first, E.stream, rec_flags);
        }
        g_prof.total_launches += 2;
    }
    cudaError_t e = launch_core(cp, E.bf16, E.greedy, E.stream);
    if (e != cudaSuccess) return cuda_fail(e, "msd_core launch");
    if (ev.first) {
        std::lock_guard<std::mutex> g(g_prof.mu);
        cudaEventRecordWithFlags(ev.second, E.stream, rec_flags);
        g_prof.pending.push_back(ev);
    }
    e = launch_tail(tp, E.bf16, E.stream);
    if (e != cudaSuccess) return cuda_fail(e, "msd_tail launch");
    return MSD_OK;
}

}  // namespace

extern "C" {

const char* msd_last_error(void) { return g_err.c_str(); }

msd_status msd_init(void) {
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    return device_init();
}
int32_t msd_abi_version(void) { return MSD_ABI_VERSION; }

size_t msd_chain_verify_workspace(int32_t L, int32_t B, int32_t K, int64_t V) {
    if (L < 2 || L > MAXL || B < 0 || K < 1 || V < 1) return 0;
    return ws_layout(L, B, K, V).total;
}
size_t msd_verify_level_workspace(int32_t B, int32_t K, int64_t V) {
    return msd_chain_verify_workspace(2, B, K, V);
}

msd_status msd_chain_verify(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                            const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                            int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                            int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                            int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                            msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                            void* stream) {
    return msd_chain_verify_proc(levels, L, B, K, V, draft_tok, u_acc, u_emit, mode, intermediate_bonus,
                                 draft_fed, n_acc, m_cand, commit_tok, commit_len, rollback, pos_dtv,
                                 pos_kl, stats, flags, ws, ws_bytes, nullptr, stream);
}

static msd_status chain_verify_impl(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                                    const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                                    int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                                    int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                                    int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                                    msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                                    const msd_processors* proc, const double* lse, void* stream) {
    float inv_temp = 1.f;
    if (proc) {
        if (!(proc->temperature > 0.f) || !(proc->temperature <= 1e6f) || !(1.f / proc->temperature <= 1e6f))
            return fail(MSD_E_ARG, "temperature %g outside (1e-6, 1e6]", (double)proc->temperature);
        if (proc->top_k != 0 || !(proc->top_p >= 1.f || proc->top_p <= 0.f))
            return fail(MSD_E_ARG, "top_k / top_p: run msd_logits_process on every level first, then pass 0 / 1 here");
        inv_temp = 1.f / proc->temperature;
    }
    if (!levels) return fail(MSD_E_ARG, "levels is NULL");
    if (L < 2 || L > MAXL) return fail(MSD_E_ARG, "L=%d outside [2,%d]", L, MAXL);
    if (B < 0 || K < 1 || K + L > MAXC) return fail(MSD_E_ARG, "bad B=%d / K=%d (need K+L <= 32)", B, K);
    if (V < 1 || V > (int64_t)128 * VS) return fail(MSD_E_ARG, "V=%lld outside [1, 524288]", (long long)V);
    if ((int64_t)L * slice_geometry(V).C > 192)
        return fail(MSD_E_ARG, "L * slices = %d * %d exceeds 192 (vocabulary too large for L levels)", L,
                    slice_geometry(V).C);
    if (mode != MSD_STOCHASTIC && mode != MSD_GREEDY) return fail(MSD_E_ARG, "unknown mode %d", mode);
    if (draft_fed < 0 || draft_fed > K) return fail(MSD_E_ARG, "draft_fed=%d outside [0,K]", draft_fed);
    if (B == 0) return MSD_OK;
    if (!draft_tok || !commit_tok || !commit_len || !flags || !n_acc)
        return fail(MSD_E_ARG, "draft_tok, n_acc, commit_tok, commit_len and flags are required");
    if (mode == MSD_STOCHASTIC && (!u_acc || !u_emit))
        return fail(MSD_E_ARG, "u_acc / u_emit are required in stochastic mode");
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    Engine E;
    memset(&E, 0, sizeof(E));
    st = validate_levels(levels, L, K, V, intermediate_bonus, -1, &E.bf16);
    if (st != MSD_OK) return st;
    for (int l = 0; l < L; ++l) {
        E.lv.ptr[l] = levels[l].ptr;
        E.lv.ld[l] = levels[l].ld;
        E.lv.bs[l] = levels[l].batch_stride;
        E.lv.rows[l] = levels[l].rows;
    }
    E.L = L; E.B = B; E.K = K; E.V = V;
    E.cand0 = draft_tok; E.m0 = nullptr;
    E.u_acc = u_acc; E.u_emit = u_emit;
    const int64_t W = K + L - 1;
    E.ua_l = (int64_t)B * W; E.ua_b = W; E.ue_l = (int64_t)B * W; E.ue_b = W;
    E.greedy = mode == MSD_GREEDY; E.ibonus = intermediate_bonus ? 1 : 0; E.fbonus = 1;
    E.draft_fed = draft_fed;
    E.n_acc = n_acc; E.m_cand = m_cand; E.out_tok = commit_tok; E.out_ld = (int32_t)W;
    E.out_len = commit_len; E.rollback = rollback;
    E.pos_dtv = pos_dtv; E.pos_kl = pos_kl; E.stats = stats; E.flags = flags;
    E.ws = ws; E.ws_bytes = ws_bytes;
    E.stream = reinterpret_cast<cudaStream_t>(stream);
    E.inv_temp = inv_temp;
    E.lse = lse;
    return run_engine(E);
}

msd_status msd_chain_verify_proc(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                                 const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                                 int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                                 int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                                 int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                                 msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                                 const msd_processors* proc, void* stream) {
    return chain_verify_impl(levels, L, B, K, V, draft_tok, u_acc, u_emit, mode, intermediate_bonus, draft_fed,
                             n_acc, m_cand, commit_tok, commit_len, rollback, pos_dtv, pos_kl, stats, flags, ws,
                             ws_bytes, proc, nullptr, stream);
}

msd_status msd_chain_verify_lse(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                                const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                                int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                                int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                                int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                                msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                                const double* lse, void* stream) {
    if (!lse) return fail(MSD_E_ARG, "lse is NULL");
    return chain_verify_impl(levels, L, B, K, V, draft_tok, u_acc, u_emit, mode, intermediate_bonus, draft_fed,
                             n_acc, m_cand, commit_tok, commit_len, rollback, pos_dtv, pos_kl, stats, flags, ws,
                             ws_bytes, nullptr, lse, stream);
}

msd_status msd_verify_level(msd_logits q, msd_logits p, int32_t B, int32_t K, int64_t V,
                            const int32_t* cand, const int32_t* m,
                            const float* u_acc, const float* u_emit,
                            int32_t mode, int32_t emit_bonus,
                            int32_t* n_acc, int32_t* out_tok, int32_t* out_len,
                            float* pos_dtv, float* pos_kl, msd_pair_stats* stats,
                            uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
    if (B < 0 || K < 1 || K + 2 > MAXC) return fail(MSD_E_ARG, "bad B=%d / K=%d (need K <= 30)", B, K);
    if (V < 1 || V > (int64_t)128 * VS) return fail(MSD_E_ARG, "V=%lld outside [1, 524288]", (long long)V);
    if ((int64_t)2 * slice_geometry(V).C > 192)
        return fail(MSD_E_ARG, "2 * slices = 2 * %d exceeds 192 (vocabulary too large)", slice_geometry(V).C);
    if (mode != MSD_STOCHASTIC && mode != MSD_GREEDY) return fail(MSD_E_ARG, "unknown mode %d", mode);
    if (B == 0) return MSD_OK;
    if (!cand || !out_tok || !out_len || !flags || !n_acc)
        return fail(MSD_E_ARG, "cand, n_acc, out_tok, out_len and flags are required");
    if (mode == MSD_STOCHASTIC && (!u_acc || !u_emit))
        return fail(MSD_E_ARG, "u_acc / u_emit are required in stochastic mode");
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    msd_logits lv[2] = {q, p};
    Engine E;
    memset(&E, 0, sizeof(E));
    st = validate_levels(lv, 2, K, V, 1, emit_bonus ? 1 : 0, &E.bf16);
    if (st != MSD_OK) return st;
    for (int l = 0; l < 2; ++l) {
        E.lv.ptr[l] = lv[l].ptr;
        E.lv.ld[l] = lv[l].ld;
        E.lv.bs[l] = lv[l].batch_stride;
        E.lv.rows[l] = lv[l].rows;
    }
    E.L = 2; E.B = B; E.K = K; E.V = V;
    E.cand0 = cand; E.m0 = m;
    E.u_acc = u_acc; E.u_emit = u_emit;
    E.ua_l = 0; E.ua_b = K; E.ue_l = 0; E.ue_b = K + 1;
    E.greedy = mode == MSD_GREEDY; E.ibonus = 0; E.fbonus = emit_bonus ? 1 : 0;
    E.draft_fed = 0;
    E.n_acc = n_acc; E.m_cand = nullptr; E.out_tok = out_tok; E.out_ld = K + 1;
    E.out_len = out_len; E.rollback = nullptr;
    E.pos_dtv = pos_dtv; E.pos_kl = pos_kl; E.stats = stats; E.flags = flags;
    E.ws = ws; E.ws_bytes = ws_bytes;
    E.stream = reinterpret_cast<cudaStream_t>(stream);
    E.inv_temp = 1.f;
    return run_engine(E);
}

msd_status msd_kv_rollback(const msd_paged_kv* kv, int32_t n_models, int32_t B,
                           const int32_t* rollback, uint32_t* flags, void* stream) {
    if (!kv || n_models < 0 || B < 0) return fail(MSD_E_ARG, "bad kv / n_models / B");
    if (n_models == 0 || B == 0) return MSD_OK;
    if (!rollback || !flags) return fail(MSD_E_ARG, "rollback and flags are required");
    for (int i = 0; i < n_models; ++i) {
        const msd_paged_kv& k = kv[i];
        if (!k.seq_len || !k.block_table || !k.free_ids || !k.free_count)
            return fail(MSD_E_ARG, "model %d: seq_len, block_table, free_ids, free_count required", i);
        if (k.block_size < 1 || k.max_blocks < 0 || k.free_cap < 0)
            return fail(MSD_E_ARG, "model %d: bad block_size / max_blocks / free_cap", i);
        if (k.cache_mask && k.mask_ld < 1) return fail(MSD_E_ARG, "model %d: mask_ld < 1", i);
    }
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    for (int m0 = 0; m0 < n_models; m0 += 8) {
        RollbackParams p;
        memset(&p, 0, sizeof(p));
        p.n_models = n_models - m0 < 8 ? n_models - m0 : 8;
        for (int i = 0; i < p.n_models; ++i) p.kv[i] = kv[m0 + i];
        p.B = B;
        p.rollback = rollback + (size_t)m0 * B;
        p.flags = flags;
        {
            std::lock_guard<std::mutex> g(g_prof.mu);
            g_prof.total_launches += 1;
        }
        cudaError_t e = launch_rollback(p, reinterpret_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_fail(e, "msd_rollback launch");
    }
    return MSD_OK;
}

msd_status msd_pool_divergence(const msd_logits* models, int32_t N, int32_t B, int32_t K, int64_t V,
                               float* pos_dtv, float* pos_kl, msd_pair_stats* stats, uint32_t* flags,
                               void* stream) {
    if (!models) return fail(MSD_E_ARG, "models is NULL");
    if (N < 2 || N > 4) return fail(MSD_E_ARG, "N=%d outside [2,4]", N);
    if (B < 0 || K < 1) return fail(MSD_E_ARG, "bad B=%d / K=%d", B, K);
    if (V < 1) return fail(MSD_E_ARG, "V=%lld < 1", (long long)V);
    if (B == 0) return MSD_OK;
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    int32_t bf16 = 0;
    st = validate_levels(models, N, K, V, 0, 0, &bf16);   // every model needs >= K rows
    if (st != MSD_OK) return st;
    PoolParams pp;
    memset(&pp, 0, sizeof(pp));
    for (int l = 0; l < N; ++l) {
        pp.lv.ptr[l] = models[l].ptr;
        pp.lv.ld[l] = models[l].ld;
        pp.lv.bs[l] = models[l].batch_stride;
        pp.lv.rows[l] = models[l].rows;
    }
    pp.N = N; pp.B = B; pp.K = K; pp.V = V;
    pp.pos_dtv = pos_dtv; pp.pos_kl = pos_kl; pp.stats = stats; pp.flags = flags;
    cudaError_t e = launch_pool(pp, bf16, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "msd_pool launch");
    return MSD_OK;
}

msd_status msd_draft_sample(const msd_logits* drafter, int32_t row, int32_t B, int64_t V,
                            const float* u, int32_t greedy, int32_t* token, float* lse,
                            float* q_tok, uint32_t* flags, void* stream) {
    if (!drafter) return fail(MSD_E_ARG, "drafter is NULL");
    if (B < 0) return fail(MSD_E_ARG, "B=%d < 0", B);
    if (V < 1 || V > (1 << 18)) return fail(MSD_E_ARG, "V=%lld outside [1, 2^18]", (long long)V);
    if (row < 0 || row >= drafter->rows) return fail(MSD_E_ARG, "row=%d outside [0, rows=%d)", row, drafter->rows);
    if (B == 0) return MSD_OK;
    if (!token) return fail(MSD_E_ARG, "token is NULL");
    if (!greedy && !u) return fail(MSD_E_ARG, "u is NULL (stochastic mode)");
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    int32_t bf16 = 0;
    st = validate_levels(drafter, 1, row + 1, V, 0, 0, &bf16);
    if (st != MSD_OK) return st;
    DraftParams dp;
    memset(&dp, 0, sizeof(dp));
    dp.z = drafter->ptr; dp.ld = drafter->ld; dp.bs = drafter->batch_stride;
    dp.row = row; dp.B = B; dp.greedy = greedy ? 1 : 0; dp.V = V;
    dp.u = u; dp.token = token; dp.lse = lse; dp.q_tok = q_tok; dp.flags = flags;
    cudaError_t e = launch_draft(dp, bf16, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "msd_draft launch");
    return MSD_OK;
}

msd_status msd_logits_process(const msd_logits* in, const msd_logits* out, int32_t B, int32_t rows, int64_t V,
                              const msd_processors* proc, float* tau, uint32_t* flags, void* stream) {
    if (!in || !out || !proc) return fail(MSD_E_ARG, "in, out and proc are required");
    if (B < 0 || rows < 1) return fail(MSD_E_ARG, "bad B=%d / rows=%d", B, rows);
    if (V < 1 || V > ((int64_t)1 << 31) - 1) return fail(MSD_E_ARG, "V=%lld outside [1, 2^31)", (long long)V);
    if (!(proc->temperature > 0.f) || !(proc->temperature <= 1e6f) || !(1.f / proc->temperature <= 1e6f))
        return fail(MSD_E_ARG, "temperature %g outside (1e-6, 1e6]", (double)proc->temperature);
    if (proc->top_k < 0) return fail(MSD_E_ARG, "top_k=%d < 0", proc->top_k);
    if (B == 0) return MSD_OK;
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    int32_t bf16 = 0, bf16o = 0;
    st = validate_levels(in, 1, rows, V, 0, 0, &bf16);
    if (st != MSD_OK) return st;
    st = validate_levels(out, 1, rows, V, 0, 0, &bf16o);
    if (st != MSD_OK) return st;
    if (bf16 != bf16o) return fail(MSD_E_DTYPE, "in and out dtypes differ");
    ProcParams pp;
    memset(&pp, 0, sizeof(pp));
    pp.in = in->ptr; pp.out = const_cast<void*>(out->ptr);
    pp.in_ld = in->ld; pp.in_bs = in->batch_stride; pp.out_ld = out->ld; pp.out_bs = out->batch_stride;
    pp.B = B; pp.rows = rows; pp.V = V;
    pp.inv_temp = 1.f / proc->temperature;
    pp.top_k = proc->top_k;
    pp.top_p = proc->top_p;
    pp.tau = tau; pp.flags = flags;
    cudaError_t e = launch_proc(pp, bf16, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "msd_proc launch");
    return MSD_OK;
}

size_t msd_lmhead_workspace(int32_t M, int64_t V) {
    if (M < 1 || V < 1) return 0;
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return lmhead_workspace(M, V, nsm > 0 ? nsm : 148);
}

msd_status msd_lmhead_lse(const void* H, const void* W, int32_t M, int32_t D, int64_t V, const int32_t* cand,
                          float* lse, float* z_cand, void* ws, size_t ws_bytes, void* stream) {
    if (M < 0 || D < 64 || D % 64 || V < 1 || V > ((int64_t)1 << 31) - 1)
        return fail(MSD_E_ARG, "bad M=%d / D=%d (multiple of 64) / V=%lld", M, D, (long long)V);
    if (M == 0) return MSD_OK;
    if (!H || !W || !lse || !ws) return fail(MSD_E_ARG, "H, W, lse and ws are required");
    if (((uintptr_t)H) % 16 || ((uintptr_t)W) % 16) return fail(MSD_E_ALIGN, "H and W must be 16-byte aligned");
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    if (ws_bytes < msd_lmhead_workspace(M, V)) return fail(MSD_E_WORKSPACE, "workspace too small");
    LmHeadParams p;
    memset(&p, 0, sizeof(p));
    p.H = H; p.W = W; p.M = M; p.D = D; p.V = V; p.cand = cand; p.lse = lse; p.z_cand = z_cand;
    p.ws = ws; p.ws_bytes = ws_bytes;
    {
        std::lock_guard<std::mutex> g(g_prof.mu);
        g_prof.total_launches += 2;
    }
    cudaError_t e = launch_lmhead(p, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "msd_lmhead launch");
    return MSD_OK;
}

msd_status msd_lmhead_logits(const void* H, const void* W, int32_t M, int32_t D, int64_t V, const int32_t* cand,
                             void* logits, int64_t ldz, double* lse64, float* z_cand, void* ws, size_t ws_bytes,
                             void* stream) {
    if (M < 0 || D < 64 || D % 64 || V < 1 || V > ((int64_t)1 << 31) - 1 || ldz < V)
        return fail(MSD_E_ARG, "bad M=%d / D=%d (multiple of 64) / V=%lld / ldz", M, D, (long long)V);
    if (M == 0) return MSD_OK;
    if (!H || !W || !logits || !lse64 || !ws) return fail(MSD_E_ARG, "H, W, logits, lse64 and ws are required");
    if (((uintptr_t)H) % 16 || ((uintptr_t)W) % 16 || ((uintptr_t)logits) % 16 || (ldz * 2) % 16)
        return fail(MSD_E_ALIGN, "H, W and the logit rows must be 16-byte aligned");
    msd_status st = check_arch();
    if (st != MSD_OK) return st;
    if (ws_bytes < msd_lmhead_workspace(M, V)) return fail(MSD_E_WORKSPACE, "workspace too small");
    LmHeadParams p;
    memset(&p, 0, sizeof(p));
    p.H = H; p.W = W; p.M = M; p.D = D; p.V = V; p.cand = cand; p.lse = nullptr; p.z_cand = z_cand;
    p.ws = ws; p.ws_bytes = ws_bytes;
    p.logits = logits; p.ldz = ldz; p.lse64 = lse64;
    {
        std::lock_guard<std::mutex> g(g_prof.mu);
        g_prof.total_launches += 2;
    }
    cudaError_t e = launch_lmhead(p, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "msd_lmhead launch");
    return MSD_OK;
}

msd_status msd_debug_set_trace(void* dev_buf, size_t bytes) {
    g_trace = reinterpret_cast<unsigned long long*>(dev_buf);
    g_trace_items = dev_buf ? bytes / 128 : 0;
    return MSD_OK;
}

msd_status msd_debug_set_knobs(int32_t pat_t, int32_t pat_r, int32_t stages, int32_t core_dbg,
                               int32_t exact_draws, double z_safe) {
    g_knobs.pat_t = pat_t;
    g_knobs.pat_r = pat_r;
    g_knobs.stages = stages;
    g_knobs.core_dbg = core_dbg;
    g_knobs.exact_draws = exact_draws ? 1 : 0;
    g_knobs.z_safe = z_safe >= 0 ? z_safe : 0.01;
    return MSD_OK;
}

msd_status msd_prof_enable(int32_t on) {
    std::lock_guard<std::mutex> g(g_prof.mu);
    g_prof.on = on != 0;
    return MSD_OK;
}

msd_status msd_prof_read(double* core_ms, int32_t* core_launches, int32_t* total_launches) {
    std::lock_guard<std::mutex> g(g_prof.mu);
    double tot = 0.0;
    for (auto& pr : g_prof.pending) {
        cudaError_t e = cudaEventSynchronize(pr.second);
        if (e != cudaSuccess) return cuda_fail(e, "msd_prof_read");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.first, pr.second);
        tot += ms;
        g_prof.pool.push_back(pr);
    }
    if (core_ms) *core_ms = tot;
    if (core_launches) *core_launches = (int32_t)g_prof.pending.size();
    if (total_launches) *total_launches = g_prof.total_launches;
    g_prof.pending.clear();
    g_prof.total_launches = 0;
    return MSD_OK;
}

}  // extern "C"
