// C-ABI core: handles, errors, the KernelTable entry points, exponent
// statistics / selection, and the CGEMM dispatcher (host orchestration of the
// device pipeline).  Mirrors reference precsel.cpp:225-322 (dispatch_cgemm),
// cgemm.cpp:25-46 (cgemm) and gemm.cpp:60-125 (mode switch).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/tcec_b200.h"
#include "tcec_handle.h"

namespace tcec {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_error(cudaError_t e, const char* what) {
    return set_error(TCEC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------ shared helpers

void stats_from_dev(const DevStats& d, int64_t n_total, tcec_exp_stats_t* s) {
    std::memset(s, 0, sizeof(*s));
    s->n1 = d.n1;
    s->n2 = d.n2;
    s->e_max_valid = d.max_bits != 0;
    s->e_max = d.max_bits ? exponent_of_bits_host(d.max_bits) : 0;
    s->n_nonzero = d.n_nonzero;
    s->n_total = uint64_t(n_total);
    s->stage2_evaluated = d.stage2_evaluated;
}

static double r1_of(const tcec_exp_stats_t* s) {
    return s->n_nonzero ? double(s->n_nonzero - s->n1) / double(s->n_nonzero) : 0.0;
}
static double r2_of(const tcec_exp_stats_t* s) {
    return s->n_nonzero ? double(s->n_nonzero - s->n2) / double(s->n_nonzero) : 0.0;
}

const char* kind_name(int kind) {
    switch (kind) {  // precsel.cpp:63-71
    case kKindFp16: return "FP16TCEC";
    case kKindFp16Scaled: return "FP16TCEC_SCALED";
    case kKindTf32: return "TF32TCEC";
    default: return "FP32_BASELINE";
    }
}

const char* forced_name(int f) {  // precsel.cpp:73-84
    static const char* names[] = {"FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC",
                                  "TF32TCEC", "FP16TCEC",    "FP16TCEC_SCALED"};
    return (f >= 0 && f <= 6) ? names[f] : "?";
}

// DecisionRecord::to_line, precsel.cpp:185-205
void format_line(char* out, size_t cap, int64_t m, int64_t n, int64_t k, const char* label,
                 int sa, int sb, const tcec_exp_stats_t* a, const tcec_exp_stats_t* b, bool has) {
    auto ratio = [&](char* buf, size_t c, const tcec_exp_stats_t* s, bool second) {
        if (!has || (second && !s->stage2_evaluated))
            std::snprintf(buf, c, "-");
        else
            std::snprintf(buf, c, "%.9g", second ? r2_of(s) : r1_of(s));
    };
    auto emax = [&](char* buf, size_t c, const tcec_exp_stats_t* s) {
        if (!has || !s->e_max_valid)
            std::snprintf(buf, c, "-");
        else
            std::snprintf(buf, c, "%d", s->e_max);
    };
    char r1a[32], r2a[32], r1b[32], r2b[32], ea[16], eb[16];
    ratio(r1a, sizeof r1a, a, false);
    ratio(r2a, sizeof r2a, a, true);
    ratio(r1b, sizeof r1b, b, false);
    ratio(r2b, sizeof r2b, b, true);
    emax(ea, sizeof ea, a);
    emax(eb, sizeof eb, b);
    std::snprintf(out, cap, "%lld,%lld,%lld,%s,%d,%d,%s,%s,%s,%s,%s,%s", (long long)m,
                  (long long)n, (long long)k, label, sa, sb, r1a, r2a, r1b, r2b, ea, eb);
}

static inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

// Host-side plan of one dispatched CGEMM (precsel.cpp:225-306 control flow)
DispatchPlan plan_dispatch(int64_t m, int64_t n, int64_t k, const tcec_dispatch_config_t& cfg) {
    DispatchPlan p;
    const int64_t mn = std::min(std::min(m, n), k);
    p.forced = cfg.force;
    if (cfg.force >= 0) {
        p.label = forced_name(cfg.force);
        switch (cfg.force) {
        case TCEC_FORCE_FP32_REF: p.tier = kTierFp32; p.kind = kKindFp32; break;
        case TCEC_FORCE_FP64_ORACLE: p.tier = kTierFp64; p.kind = kKindFp32; break;
        case TCEC_FORCE_TF32_TC: p.tier = kTierTc; p.kind = kKindTf32; p.corrected = 0; break;
        case TCEC_FORCE_FP16_TC: p.tier = kTierTc; p.kind = kKindFp16; p.corrected = 0; break;
        case TCEC_FORCE_TF32_TCEC: p.tier = kTierTc; p.kind = kKindTf32; break;
        case TCEC_FORCE_FP16_TCEC: p.tier = kTierTc; p.kind = kKindFp16; break;
        case TCEC_FORCE_FP16_TCEC_SCALED:
            p.tier = kTierTc;
            p.kind = -1;  // scales from statistics (precsel.cpp:264-271)
            p.stats = true;
            p.forced_scaled = true;
            p.kind_known = kKindFp16Scaled;
            break;
        default: p.tier = kTierInvalid; break;
        }
    } else if (mn >= cfg.size_auto) {
        p.tier = kTierTc;
        p.kind = -1;  // decided on the device
        p.stats = true;
    } else if (mn >= cfg.size_tf32) {
        p.tier = kTierTc;
        p.kind = kKindTf32;
        p.label = kind_name(kKindTf32);
    } else {
        p.tier = kTierFp32;
        p.kind = kKindFp32;
        p.label = kind_name(kKindFp32);
    }
    if (p.kind >= 0 && p.tier == kTierTc) p.kind_known = p.kind;
    if (p.tier == kTierFp32 || p.tier == kTierFp64) p.kind_known = kKindFp32;
    p.kp = round_up(2 * k, 64);
    return p;
}

size_t plan_workspace(const DispatchPlan& p, int64_t m, int64_t n) {
    if (p.tier != kTierTc) return 0;
    const int elem = (p.kind == kKindFp16 || p.forced_scaled) ? 2 : 4;  // auto: sized for tf32
    // room for either operand layout: B-expanded (m + 2n rows) or A-expanded (2m + n)
    auto planes = [&](int64_t ra, int64_t rb) {
        return 2 * round_up(int64_t(size_t(ra) * p.kp * elem), 1024) +
               2 * round_up(int64_t(size_t(rb) * p.kp * elem), 1024);
    };
    return size_t(std::max(planes(m, 2 * n), planes(2 * m, n)));
}

// Operand layout of a tensor-core dispatch: the complex block expansion goes to
// the smaller operand (A-expanded when m < n), unless the handle forces one.
bool use_xa(const Handle& h, int64_t m, int64_t n) {
    if (h.layout == 1) return false;
    if (h.layout == 2) return true;
    return m < n && h.gemm_pair != kVariantPair;
}

// Operand planes in the workspace + the GEMM arguments of a tensor-core dispatch.
TcecGemmArgs tc_gemm_args(const Handle& h, const DispatchPlan& p, void* ws, float* c, int64_t m,
                          int64_t n, DevDecision* d, bool allow_xa) {
    const int elem = (p.kind == kKindFp16 || p.forced_scaled) ? 2 : 4;
    const bool xa = allow_xa && use_xa(h, m, n);
    const int64_t rows_a = xa ? 2 * m : m, rows_b = xa ? n : 2 * n;  // GEMM M and N
    const size_t abytes = round_up(int64_t(size_t(rows_a) * p.kp * elem), 1024);
    const size_t bbytes = round_up(int64_t(size_t(rows_b) * p.kp * elem), 1024);
    uint8_t* w = static_cast<uint8_t*>(ws);
    TcecGemmArgs g{};
    g.a_hi = w;
    g.a_lo = w + abytes;
    g.b_hi = w + 2 * abytes;
    g.b_lo = w + 2 * abytes + bbytes;
    g.c = c;
    g.m = rows_a;
    g.a_rows = rows_a;
    g.n2 = rows_b;
    g.kp = p.kp;
    g.xa = xa ? 1 : 0;
    g.d = d;
    g.kind_fixed = p.kind;
    g.corrected = p.corrected;
    // TF32 flush interval (its own 32-element k-blocks) in the high half;
    // TCEC_TF32_FLUSH overrides it (0 = as many k-blocks as FP16)
    static const int tf32_flush = [] {
        const char* e = std::getenv("TCEC_TF32_FLUSH");
        return e ? std::max(0, std::min(64, std::atoi(e))) : 0;
    }();
    g.flush_kblocks = p.corrected ? (h.flush_kblocks | (h.flush_kblocks > 0 ? tf32_flush << 16 : 0)) : 0;
    // no A-expanded 256x128 pair kernel; the host-buffer pipeline (allow_xa =
    // false) needs a kernel that takes row chunks and column blocks
    g.pair = resolve_gemm_variant(h.gemm_pair, rows_a, rows_b, p.kp, h.sm_count, !xa && allow_xa, allow_xa);
    g.sms = h.sm_count;
    g.fmt = (p.kind < 0 && !p.forced_scaled) ? -1  // format chosen by the device decision
                                             : (p.kind == kKindTf32 ? kTf32 : kFp16);
    return g;
}

// GEMM of rows [r0, r1) of A' (chunked: no split-K, so a chunk computes
// exactly what the whole launch would), then the hook's done() on the C rows
// they produce (A-expanded layout: GEMM rows 2i, 2i+1 -> C row i; r0 even, and
// C row r0 / 2 starts at float r0 * n2 = r0 / 2 * 2n in both layouts)
int launch_gemm_rows(const TcecGemmArgs& g, int64_t r0, int64_t r1, bool chunked,
                     const ChunkHook* hook, cudaStream_t s) {
    TcecGemmArgs gc = g;
    gc.no_split = chunked;
    gc.m = r1 - r0;
    gc.a_row_off = r0;
    gc.c = g.c + r0 * g.n2;
    const int e = launch_tcec_gemm(gc, s);
    if (e) return cuda_error(cudaError_t(e), g.fmt < 0 ? "tcec_gemm auto"
                                             : (g.fmt == kTf32 ? "tcec_gemm tf32" : "tcec_gemm f16"));
    if (hook && hook->done) return g.xa ? hook->done(hook->ctx, r0 / 2, r1 / 2) : hook->done(hook->ctx, r0, r1);
    return TCEC_OK;
}

// Launch the device pipeline of one dispatch (no host synchronization).
int launch_dispatch(Handle& h, const float* a, const float* b, float* c, int64_t m, int64_t n,
                    int64_t k, const tcec_dispatch_config_t& cfg, const DispatchPlan& p,
                    DevDecision* d, void* ws, const ChunkHook* hook, const MatrixView* va,
                    const MatrixView* vb) {
    cudaStream_t s = h.stream;
    if (p.tier == kTierInvalid) return set_error(TCEC_ERR_INVALID_ARGUMENT, "unknown forced mode");
    if ((va || vb) && (p.tier != kTierTc || hook))
        return set_error(TCEC_ERR_LOGIC, "operand views need the tensor-core tier");
    if (p.tier == kTierTc && cfg.k_tile < 1)
        return set_error(TCEC_ERR_INVALID_ARGUMENT, "k_tile must be >= 1");
    const bool prof = h.prof && h.ev[0];
    if (prof) cudaEventRecord(h.ev[0], s);
    // only the tensor-core tier writes the decision slot (finish_dispatch reads
    // nothing from it for the SIMT tiers)
    if (p.tier == kTierTc) cudaMemsetAsync(d, 0, sizeof(DevDecision), s);
    if (p.stats) {
        launch_stats1(a, 2 * m * k, b, 2 * k * n, d, s);
        const double t = p.forced_scaled ? 1.0 : cfg.threshold_t;
        launch_stats2(a, 2 * m * k, b, 2 * k * n, d, t, cfg.target_max_exponent, 0, s, 1, cfg.threshold_t,
                      p.forced_scaled ? 1 : 0);
    }
    if (prof) cudaEventRecord(h.ev[1], s);
    if (m == 0 || n == 0 || k == 0 || p.tier != kTierTc) {
        if (prof) cudaEventRecord(h.ev[2], s);
    }
    if (m == 0 || n == 0) {
        if (prof) cudaEventRecord(h.ev[3], s);
        return TCEC_OK;
    }
    if (k == 0) {
        // every mode yields +0 (the reference chains start at 0.0f)
        cudaMemsetAsync(c, 0, size_t(m) * n * 8, s);
        if (prof) cudaEventRecord(h.ev[3], s);
        return TCEC_OK;
    }
    switch (p.tier) {
    case kTierFp32:
        launch_cgemm_fp32_ref(reinterpret_cast<const float2*>(a), reinterpret_cast<const float2*>(b),
                              reinterpret_cast<float2*>(c), m, n, k, s);
        if (prof) cudaEventRecord(h.ev[3], s);
        return hook && hook->done ? hook->done(hook->ctx, 0, m) : TCEC_OK;
    case kTierFp64:
        launch_cgemm_fp64(reinterpret_cast<const float2*>(a), reinterpret_cast<const float2*>(b),
                          reinterpret_cast<float2*>(c), m, n, k, s);
        if (prof) cudaEventRecord(h.ev[3], s);
        return hook && hook->done ? hook->done(hook->ctx, 0, m) : TCEC_OK;
    default: break;
    }
    // tensor-core tier: operand preparation + tcgen05 GEMM(s)
    TcecGemmArgs g = tc_gemm_args(h, p, ws, c, m, n, d, true);
    void* ahi = const_cast<void*>(g.a_hi);
    void* alo = const_cast<void*>(g.a_lo);
    void* bhi = const_cast<void*>(g.b_hi);
    void* blo = const_cast<void*>(g.b_lo);
    if (g.xa) {
        launch_prep_ax(a, m, k, p.kp, ahi, alo, d, p.kind, p.corrected, s, va);
        launch_prep_bx(b, k, n, p.kp, bhi, blo, d, p.kind, p.corrected, s, vb);
    } else {
        launch_prep_a(a, m, k, p.kp, ahi, alo, d, p.kind, p.corrected, s, 0, va);
        launch_prep_b(b, k, n, p.kp, bhi, blo, d, p.kind, p.corrected, s, 0, vb);
    }
    if (prof) cudaEventRecord(h.ev[2], s);
    // row chunks (host-buffer API): only the wide kernel indexes into A' by row
    int chunks = hook ? std::max(1, hook->chunks) : 1;
    if (g.pair != kVariantWide && g.pair != kVariantWideMc) chunks = 1;
    const int64_t gm = g.m;  // GEMM rows (2m in the A-expanded layout)
    const int64_t rows_per = round_up((gm + chunks - 1) / chunks, 256);
    for (int64_t r0 = 0; r0 < gm; r0 += rows_per) {
        const int64_t r1 = std::min(gm, r0 + rows_per);
        const int rc = launch_gemm_rows(g, r0, r1, chunks > 1, hook, s);
        if (rc) return rc;
    }
    if (prof) cudaEventRecord(h.ev[3], s);
    return TCEC_OK;
}

// Fill a host result from the (already copied back) device decision.
int finish_dispatch(const DispatchPlan& p, const DevDecision& dd, int64_t m, int64_t n, int64_t k,
                    tcec_dispatch_result_t* res) {
    std::memset(res, 0, sizeof(*res));
    if (p.stats) {
        res->has_stats = 1;
        stats_from_dev(dd.st[0], 2 * m * k, &res->stats_a);
        stats_from_dev(dd.st[1], 2 * k * n, &res->stats_b);
    }
    int kind = p.stats ? dd.kind : p.kind_known;
    if (p.forced >= 0) {
        // forced-mode decisions, precsel.cpp:238-272
        static const int forced_kind[] = {kKindFp32, kKindFp32, kKindTf32, kKindFp16,
                                          kKindTf32, kKindFp16, kKindFp16Scaled};
        kind = forced_kind[p.forced];
    }
    if (kind < 0)
        return set_error(TCEC_ERR_LOGIC, "matrix_tolerance: stage-2 statistics required but skipped");
    res->kind = kind;
    if (kind == kKindFp16Scaled) {
        res->scale_a = dd.scale_a;
        res->scale_b = dd.scale_b;
    }
    const bool dev_written = p.tier == kTierTc;
    res->overflow = dev_written && dd.overflow ? 1 : 0;
    const char* label = p.forced >= 0 ? forced_name(p.forced) : kind_name(kind);
    format_line(res->line, sizeof res->line, m, n, k, label, res->scale_a, res->scale_b,
                &res->stats_a, &res->stats_b, res->has_stats != 0);
    if (dev_written && dd.scale_overflow)
        return set_error(TCEC_ERR_SCALE_OVERFLOW, "scaled component left the f32 range");
    return TCEC_OK;
}

}  // namespace tcec

using namespace tcec;

// Captured dispatch graphs bake in the workspace / decision addresses (and the
// pinned decision mirror their D2H copy targets); any reallocation retires them.
void tcec_handle_s::drop_graphs() {
    for (auto& g : graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g = DispatchGraph{};
    }
    n_graphs = 0;
    next_graph = 0;
}

void* tcec_handle_s::workspace(size_t bytes) {
    if (bytes <= ws_bytes) return ws;
    cudaStreamSynchronize(stream);
    drop_graphs();
    if (ws) cudaFree(ws);
    ws = nullptr;
    ws_bytes = 0;
    size_t want = bytes + bytes / 4 + (1u << 20);
    if (cudaMalloc(&ws, want) != cudaSuccess) {
        cudaGetLastError();
        if (cudaMalloc(&ws, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        want = bytes;
    }
    ws_bytes = want;
    return ws;
}

tcec::DevDecision* tcec_handle_s::decisions(int slots) {
    if (slots <= dec_slots) return dec;
    cudaStreamSynchronize(stream);
    drop_graphs();
    if (dec) cudaFree(dec);
    if (dec_host) cudaFreeHost(dec_host);
    dec = nullptr;
    dec_host = nullptr;
    dec_slots = 0;
    const int want = slots < 16 ? 16 : slots;
    if (cudaMalloc(&dec, sizeof(tcec::DevDecision) * want) != cudaSuccess) return nullptr;
    if (cudaMallocHost(&dec_host, sizeof(tcec::DevDecision) * want) != cudaSuccess) return nullptr;
    // slots of SIMT-tier steps are never written by a kernel but are read back
    // with the others (contraction logs): start them defined
    if (cudaMemset(dec, 0, sizeof(tcec::DevDecision) * want) != cudaSuccess) return nullptr;
    std::memset(dec_host, 0, sizeof(tcec::DevDecision) * want);
    dec_slots = want;
    return dec;
}

tcec_handle_s::~tcec_handle_s() {
    if (stream) cudaStreamSynchronize(stream);
    stage.reset();
    if (ws) cudaFree(ws);
    if (io) cudaFree(io);
    if (dec) cudaFree(dec);
    if (dec_host) cudaFreeHost(dec_host);
    if (scratch_host) cudaFreeHost(scratch_host);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (in_stream) cudaStreamDestroy(in_stream);
    if (gemm_stream2) cudaStreamDestroy(gemm_stream2);
    for (auto& e : in_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : chunk_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : batch_ev)
        if (e) cudaEventDestroy(e);
    for (auto& g : graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
}


#define CHECK_HANDLE(h)                                                         \
    do {                                                                        \
        if (!(h)) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null handle");   \
        cudaSetDevice((h)->device);                                             \
    } while (0)

#define CUDA_TRY(expr)                                                          \
    do {                                                                        \
        cudaError_t e_ = (expr);                                                \
        if (e_ != cudaSuccess) return cuda_error(e_, #expr);                    \
    } while (0)

extern "C" {

const char* tcec_last_error(void) { return g_last_error.c_str(); }

const char* tcec_version(void) {
    return "tcec_b200 sm_100a: tcgen05 TCEC CGEMM (f16/tf32, TMEM main+corr, RN flush), "
           "device-side precision selection, bit-exact SIMT FP32/FP64 tiers";
}

int tcec_create(int device, tcec_handle* out) {
    if (!out) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return set_error(TCEC_ERR_CUDA, "no CUDA device (the TCEC path has no CPU fallback)");
    }
    if (device < 0 || device >= count) return set_error(TCEC_ERR_INVALID_ARGUMENT, "bad device");
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_error(TCEC_ERR_CUDA, std::string("sm_100 required, found ") + prop.name);
    CUDA_TRY(cudaSetDevice(device));
    auto* h = new tcec_handle_s();
    h->device = device;
    h->sm_count = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete h;
        return set_error(TCEC_ERR_CUDA, "stream creation failed");
    }
    h->stream = h->own_stream;
    {
        // contraction intermediates are stream-ordered allocations of up to
        // GiBs; keep freed blocks in the pool across synchronizations instead
        // of returning them to the OS (re-mapping them per slice / bitstring
        // cost more than the kernels)
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = ~uint64_t(0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    if (!h->decisions(64)) {
        delete h;
        return set_error(TCEC_ERR_CUDA, "decision buffer allocation failed");
    }
    if (cudaMallocHost(&h->scratch_host, 4096) != cudaSuccess) {
        delete h;
        return set_error(TCEC_ERR_CUDA, "pinned scratch allocation failed");
    }
    *out = h;
    return TCEC_OK;
}

int tcec_destroy(tcec_handle h) {
    if (!h) return TCEC_OK;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    delete h;
    return TCEC_OK;
}

int tcec_set_stream(tcec_handle h, void* stream) {
    CHECK_HANDLE(h);
    h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
    return TCEC_OK;
}

void* tcec_get_stream(tcec_handle h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int tcec_synchronize(tcec_handle h) {
    CHECK_HANDLE(h);
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return TCEC_OK;
}

int tcec_set_flush_kblocks(tcec_handle h, int kblocks) {
    CHECK_HANDLE(h);
    if (kblocks < 0) return set_error(TCEC_ERR_INVALID_ARGUMENT, "flush interval must be >= 0");
    h->flush_kblocks = kblocks;
    return TCEC_OK;
}

int tcec_get_flush_kblocks(tcec_handle h) { return h ? h->flush_kblocks : -1; }

int tcec_set_executor(tcec_handle h, int policy) {
    CHECK_HANDLE(h);
    if (policy < 0 || policy > 3) return set_error(TCEC_ERR_INVALID_ARGUMENT, "executor must be 0..3");
    h->executor = policy;
    return TCEC_OK;
}

int tcec_set_gemm_variant(tcec_handle h, int variant) {
    CHECK_HANDLE(h);
    if (variant < 0 || variant > 6) return set_error(TCEC_ERR_INVALID_ARGUMENT, "variant must be 0..6");
    h->gemm_pair = variant;
    return TCEC_OK;
}

int tcec_set_operand_layout(tcec_handle h, int layout) {
    CHECK_HANDLE(h);
    if (layout < 0 || layout > 2) return set_error(TCEC_ERR_INVALID_ARGUMENT, "layout must be 0..2");
    h->layout = layout;
    return TCEC_OK;
}

int tcec_get_operand_layout(tcec_handle h) { return h ? h->layout : -1; }

int tcec_profile_enable(tcec_handle h, int on) {
    CHECK_HANDLE(h);
    if (on && !h->ev[0])
        for (auto& e : h->ev) CUDA_TRY(cudaEventCreate(&e));
    if (on && !h->batch_ev[0])
        for (auto& e : h->batch_ev) CUDA_TRY(cudaEventCreate(&e));
    h->prof = on != 0;
    h->prof_ms[0] = h->prof_ms[1] = h->prof_ms[2] = 0.0;
    h->prof_count = 0;
    h->batch_ms = 0.0;
    h->batch_count = 0;
    return TCEC_OK;
}

int tcec_profile_read_batches(tcec_handle h, double* ms, int64_t* count) {
    CHECK_HANDLE(h);
    if (ms) *ms = h->batch_ms;
    if (count) *count = h->batch_count;
    return TCEC_OK;
}

int tcec_host_pipeline_stats(tcec_handle h, int64_t* runs, int64_t* reruns) {
    CHECK_HANDLE(h);
    if (runs) *runs = h->pipe_runs;
    if (reruns) *reruns = h->pipe_reruns;
    return TCEC_OK;
}

int tcec_profile_read(tcec_handle h, double* stage_ms, int64_t* count) {
    CHECK_HANDLE(h);
    for (int i = 0; i < 3; ++i) stage_ms[i] = h->prof_ms[i];
    if (count) *count = h->prof_count;
    return TCEC_OK;
}

// ------------------------------------------------------------ KernelTable

static int read_flag(tcec_handle h, unsigned* dflag, int* out) {
    unsigned* hf = static_cast<unsigned*>(h->scratch_host);
    CUDA_TRY(cudaMemcpyAsync(hf, dflag, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (out && *hf) *out = 1;
    return TCEC_OK;
}

int tcec_quantize_buf(tcec_handle h, const float* src, float* dst, int64_t n, int fmt,
                      int rounding, int* overflow) {
    CHECK_HANDLE(h);
    if (fmt < 0 || fmt > 1 || rounding < 0 || rounding > 1)
        return set_error(TCEC_ERR_INVALID_ARGUMENT, "bad format or rounding");
    DevDecision* d = h->dec;
    CUDA_TRY(cudaMemsetAsync(&d->overflow, 0, sizeof(unsigned), h->stream));
    launch_quantize(src, dst, n, fmt, rounding, &d->overflow, h->stream);
    CUDA_TRY(cudaGetLastError());
    return read_flag(h, &d->overflow, overflow);
}

int tcec_split_buf(tcec_handle h, const float* src, float* hi, float* lo, int64_t n, int fmt,
                   int* overflow) {
    CHECK_HANDLE(h);
    if (fmt < 0 || fmt > 1) return set_error(TCEC_ERR_INVALID_ARGUMENT, "bad format");
    DevDecision* d = h->dec;
    CUDA_TRY(cudaMemsetAsync(&d->overflow, 0, sizeof(unsigned), h->stream));
    launch_split_flat(src, hi, lo, n, fmt, &d->overflow, h->stream);
    CUDA_TRY(cudaGetLastError());
    return read_flag(h, &d->overflow, overflow);
}

int tcec_scale_buf(tcec_handle h, const float* src, float* dst, int64_t n, int scale_exp) {
    CHECK_HANDLE(h);
    launch_scale(src, dst, n, scale_exp, nullptr, h->stream);
    CUDA_TRY(cudaGetLastError());
    return TCEC_OK;
}

int tcec_add_buf(tcec_handle h, const float* a, const float* b, float* dst, int64_t n) {
    CHECK_HANDLE(h);
    launch_add_sub(a, b, dst, n, 0, h->stream);
    CUDA_TRY(cudaGetLastError());
    return TCEC_OK;
}

int tcec_sub_buf(tcec_handle h, const float* a, const float* b, float* dst, int64_t n) {
    CHECK_HANDLE(h);
    launch_add_sub(a, b, dst, n, 1, h->stream);
    CUDA_TRY(cudaGetLastError());
    return TCEC_OK;
}

int tcec_scale_components(tcec_handle h, float* x, int64_t n, int scale_exp, int check) {
    CHECK_HANDLE(h);
    DevDecision* d = h->dec;
    CUDA_TRY(cudaMemsetAsync(&d->scale_overflow, 0, sizeof(unsigned), h->stream));
    launch_scale(x, x, n, scale_exp, check ? &d->scale_overflow : nullptr, h->stream);
    CUDA_TRY(cudaGetLastError());
    if (!check) return TCEC_OK;
    int bad = 0;
    const int rc = read_flag(h, &d->scale_overflow, &bad);
    if (rc) return rc;
    if (bad) return set_error(TCEC_ERR_SCALE_OVERFLOW, "scaled component left the f32 range");
    return TCEC_OK;
}

// Test hook for the hot-path operand preparation (prep_a / prep_b): the same
// kernels launch_dispatch runs, for a decision fixed by the caller, writing
// straight into caller planes so a test can compare them bit for bit with the
// reference's split_buf(scale_buf(x)) (kernels_scalar.cpp:24-40).
int64_t tcec_prep_kp(int64_t k) { return round_up(2 * k, 64); }

int tcec_debug_prep(tcec_handle h, const void* a, const void* b, int64_t m, int64_t n, int64_t k,
                    int kind, int scale_a, int scale_b, int corrected, void* a_hi, void* a_lo,
                    void* b_hi, void* b_lo, int* flags) {
    return tcec_debug_prep_layout(h, a, b, m, n, k, kind, scale_a, scale_b, corrected, 0, a_hi, a_lo,
                                  b_hi, b_lo, flags);
}

int tcec_debug_prep_layout(tcec_handle h, const void* a, const void* b, int64_t m, int64_t n, int64_t k,
                           int kind, int scale_a, int scale_b, int corrected, int xa, void* a_hi,
                           void* a_lo, void* b_hi, void* b_lo, int* flags) {
    CHECK_HANDLE(h);
    if (m < 0 || n < 0 || k < 0) return set_error(TCEC_ERR_SHAPE_MISMATCH, "negative extent");
    if (kind != kKindFp16 && kind != kKindFp16Scaled && kind != kKindTf32)
        return set_error(TCEC_ERR_INVALID_ARGUMENT, "debug_prep: kind must be a tensor-core kind");
    DevDecision* d = h->decisions(1);
    if (!d) return set_error(TCEC_ERR_CUDA, "decision buffer allocation failed");
    DevDecision* hd = h->dec_host;
    std::memset(hd, 0, sizeof(DevDecision));
    hd->kind = kind;
    hd->scale_a = scale_a;
    hd->scale_b = scale_b;
    CUDA_TRY(cudaMemcpyAsync(d, hd, sizeof(DevDecision), cudaMemcpyHostToDevice, h->stream));
    const int64_t kp = tcec_prep_kp(k);
    const int cr = corrected ? 1 : 0;
    if (a && m > 0 && k > 0) {
        if (xa)
            launch_prep_ax(static_cast<const float*>(a), m, k, kp, a_hi, a_lo, d, -1, cr, h->stream);
        else
            launch_prep_a(static_cast<const float*>(a), m, k, kp, a_hi, a_lo, d, -1, cr, h->stream, 0);
    }
    if (b && n > 0 && k > 0) {
        if (xa)
            launch_prep_bx(static_cast<const float*>(b), k, n, kp, b_hi, b_lo, d, -1, cr, h->stream);
        else
            launch_prep_b(static_cast<const float*>(b), k, n, kp, b_hi, b_lo, d, -1, cr, h->stream, 0);
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(hd, d, sizeof(DevDecision), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (flags) {
        flags[0] = hd->overflow ? 1 : 0;
        flags[1] = hd->scale_overflow ? 1 : 0;
    }
    return TCEC_OK;
}

// ------------------------------------------------------ statistics / selection

int tcec_exp_stats(tcec_handle h, const void* x, int64_t rows, int64_t cols, int target,
                   int staged, double t, tcec_exp_stats_t* out) {
    CHECK_HANDLE(h);
    if (!out) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null output");
    DevDecision* d = h->dec;
    const int64_t n = 2 * rows * cols;
    const float* p = static_cast<const float*>(x);
    CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(DevDecision), h->stream));
    launch_stats1(p, n, nullptr, 0, d, h->stream);
    launch_stats2(p, n, nullptr, 0, d, t, target, staged ? 0 : 1, h->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h->dec_host, d, sizeof(DevDecision), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    DevStats st = h->dec_host->st[0];
    // finalize exactly as precsel.cpp:95-104
    tcec_exp_stats_t s;
    stats_from_dev(st, n, &s);
    bool pass = true;
    if (s.n_nonzero != 0) {
        const double r1 = r1_of(&s);
        pass = !(r1 > t) && (!s.e_max_valid || s.e_max <= target);
    }
    if (staged && pass) {
        s.n2 = s.n1;
        s.stage2_evaluated = 0;
    } else {
        s.stage2_evaluated = 1;
        if (!s.e_max_valid) s.n2 = 0;
    }
    *out = s;
    return TCEC_OK;
}

double tcec_r1(const tcec_exp_stats_t* s) { return r1_of(s); }
double tcec_r2(const tcec_exp_stats_t* s) { return r2_of(s); }

int tcec_matrix_tolerance(const tcec_exp_stats_t* s, double t, int target, int* level) {
    // precsel.cpp:106-121
    if (!s || !level) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (s->n_nonzero == 0) {
        *level = 2;
        return TCEC_OK;
    }
    const bool pass = !(r1_of(s) > t) && (!s->e_max_valid || s->e_max <= target);
    if (pass) {
        *level = 2;
        return TCEC_OK;
    }
    if (!s->stage2_evaluated)
        return set_error(TCEC_ERR_LOGIC, "matrix_tolerance: stage-2 statistics required but skipped");
    *level = r2_of(s) <= t ? 1 : 0;
    return TCEC_OK;
}

int tcec_select_mode(int la, int eva, int ea, int lb, int evb, int eb, int target, int* kind,
                     int* sa, int* sb) {
    // precsel.cpp:123-135
    if (!kind || !sa || !sb) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    *sa = *sb = 0;
    if (la == 2 && lb == 2) {
        *kind = kKindFp16;
    } else if (la >= 1 && lb >= 1) {
        *kind = kKindFp16Scaled;
        *sa = eva ? target - ea : 0;
        *sb = evb ? target - eb : 0;
    } else {
        *kind = kKindTf32;
    }
    return TCEC_OK;
}

// ------------------------------------------------------------------ CGEMM

void tcec_default_config(tcec_dispatch_config_t* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->threshold_t = 0.0;  // SelectionPolicy defaults, precsel.hpp:60-65
    cfg->size_auto = 2048;
    cfg->size_tf32 = 512;
    cfg->target_max_exponent = 14;
    cfg->k_tile = 16;        // TilingConfig, gemm.hpp:28-30
    cfg->force = -1;
}

int tcec_cgemm(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
               int64_t k, int mode, int k_tile, int* overflow) {
    CHECK_HANDLE(h);
    static const int mode_to_force[] = {TCEC_FORCE_FP32_REF, TCEC_FORCE_FP64_ORACLE,
                                        TCEC_FORCE_TF32_TC,  TCEC_FORCE_FP16_TC,
                                        TCEC_FORCE_TF32_TCEC, TCEC_FORCE_FP16_TCEC};
    if (mode < 0 || mode > 5) return set_error(TCEC_ERR_INVALID_ARGUMENT, "unknown GEMM mode");
    tcec_dispatch_config_t cfg;
    tcec_default_config(&cfg);
    cfg.k_tile = k_tile;
    cfg.force = mode_to_force[mode];
    tcec_dispatch_result_t res;
    const int rc = tcec_dispatch_cgemm(h, a, b, c, m, n, k, &cfg, &res);
    if (rc == TCEC_OK && overflow && res.overflow) *overflow = 1;
    return rc;
}

int tcec_dispatch_cgemm(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
                        int64_t k, const tcec_dispatch_config_t* cfg, tcec_dispatch_result_t* res) {
    CHECK_HANDLE(h);
    if (!cfg || !res) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (m < 0 || n < 0 || k < 0) return set_error(TCEC_ERR_SHAPE_MISMATCH, "negative extent");
    const DispatchPlan p = plan_dispatch(m, n, k, *cfg);
    void* ws = nullptr;
    const size_t wsb = plan_workspace(p, m, n);
    if (wsb) {
        ws = h->workspace(wsb);
        if (!ws) return set_error(TCEC_ERR_CUDA, "workspace allocation failed");
    }
    DevDecision* d = h->dec;
    // small problems are bound by the host enqueue of their ~7 operations:
    // replay a captured graph of the whole sequence when the same pointers,
    // shape and configuration come again (kernels read the data at run time)
    const bool small = double(m) * double(n) * double(k) <= 8.6e9 && m > 0 && n > 0 && k > 0 &&
                       !(h->prof && h->ev[0]);
    Handle::DispatchGraph key{a, b, c, ws, d, m, n, k, cfg->threshold_t, cfg->size_auto,
                              cfg->size_tf32, cfg->target_max_exponent, cfg->k_tile, cfg->force,
                              h->gemm_pair, h->flush_kblocks, h->layout, h->stream, nullptr};
    auto same = [&](const Handle::DispatchGraph& g) {
        return g.a == key.a && g.b == key.b && g.c == key.c && g.ws == key.ws && g.dec == key.dec &&
               g.m == m && g.n == n && g.k == k && g.t == key.t && g.size_auto == key.size_auto &&
               g.size_tf32 == key.size_tf32 && g.target == key.target && g.k_tile == key.k_tile &&
               g.force == key.force && g.variant == key.variant && g.flush == key.flush &&
               g.layout == key.layout && g.stream == key.stream;
    };
    const Handle::DispatchGraph* hit = nullptr;
    if (small)
        for (int i = 0; i < h->n_graphs; ++i)
            if (same(h->graphs[i])) hit = &h->graphs[i];
    if (!hit && small) {
        // capture once; on any capture problem fall through to direct launches
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            int rc = launch_dispatch(*h, static_cast<const float*>(a), static_cast<const float*>(b),
                                     static_cast<float*>(c), m, n, k, *cfg, p, d, ws);
            if (rc == TCEC_OK)
                cudaMemcpyAsync(h->dec_host, d, sizeof(DevDecision), cudaMemcpyDeviceToHost, h->stream);
            const cudaError_t ec = cudaStreamEndCapture(h->stream, &graph);
            cudaGraphExec_t exec = nullptr;
            if (rc == TCEC_OK && ec == cudaSuccess && graph &&
                cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
                Handle::DispatchGraph& slot = h->graphs[h->next_graph];
                if (slot.exec) cudaGraphExecDestroy(slot.exec);
                slot = key;
                slot.exec = exec;
                h->next_graph = (h->next_graph + 1) % 8;
                h->n_graphs = std::min(8, h->n_graphs + 1);
                hit = &slot;
            }
            if (graph) cudaGraphDestroy(graph);
            // a capture that failed for any reason falls through to direct
            // launches, which report a genuine error themselves
            if (!hit) cudaGetLastError();
        } else {
            cudaGetLastError();
        }
    }
    if (hit) {
        CUDA_TRY(cudaGraphLaunch(hit->exec, h->stream));
    } else {
        int rc = launch_dispatch(*h, static_cast<const float*>(a), static_cast<const float*>(b),
                                 static_cast<float*>(c), m, n, k, *cfg, p, d, ws);
        if (rc) return rc;
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(h->dec_host, d, sizeof(DevDecision), cudaMemcpyDeviceToHost, h->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (h->prof && h->ev[0]) {
        for (int i = 0; i < 3; ++i) {
            float ms = 0.0f;
            if (cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]) == cudaSuccess) h->prof_ms[i] += ms;
        }
        ++h->prof_count;
    }
    return finish_dispatch(p, *h->dec_host, m, n, k, res);
}

// Host-buffer pipeline of a large tensor-core dispatch (m >= 8192, wide
// kernel).  Operands go up on in_stream as column parts of B (packed part by
// part into the staging buffer) and row chunks of A, in the order
// B[front parts], A[0..], B[back parts]; every (A chunk, B column block) GEMM
// starts as soon as both have landed, and each finished block of C goes back
// on copy_stream -- the PCIe transfers overlap the tensor-core work instead of
// preceding it (16384^3: the GEMM starts after ~1/2 of B and 1/12 of A instead
// of all of B).  GEMM blocks alternate between two streams so one block's
// tail overlaps the next block's start.
//
// The precision decision needs statistics of all of A and B, which land last:
// the blocks therefore run under a decision taken from the front parts of B
// and the first chunk of A (slot 1); the exact decision over everything (slot
// 0) follows, and the caller checks that the two agree in everything prep and
// GEMM read (kind, scales, the selection-stage flags).  On disagreement the
// plain path reruns (tcec_dispatch_cgemm_host), so the result is always the
// one the unpipelined dispatch produces.  Statistics are order-free counts and
// maxima, so the part-packed staging of B yields the same statistics.
struct HostPipe {
    int nch = 1, q = 1, front = 1;
    int64_t rows_per = 0, wq = 0;
};

// TCEC_HOST_SPEC_TF32=0: take the sample's decision as is (A/B)
static bool host_spec_tf32() {
    static const bool on = [] {
        const char* e = std::getenv("TCEC_HOST_SPEC_TF32");
        return !(e && e[0] == '0');
    }();
    return on;
}

static HostPipe plan_host_pipe(int64_t m, int64_t n, int chunks, int parts) {
    HostPipe hp;
    // >= 1024-row chunks: smaller GEMM blocks (at m < 16384) leave SMs idle
    static const int64_t min_rows = [] {
        const char* e = std::getenv("TCEC_HOST_MINROWS");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? int64_t(v) : int64_t(1024);
    }();
    hp.rows_per = std::max(round_up((m + chunks - 1) / chunks, 256), round_up(std::min(m, min_rows), 256));
    hp.nch = int((m + hp.rows_per - 1) / hp.rows_per);
    hp.q = int(std::max<int64_t>(1, std::min<int64_t>(parts, n / 256)));  // parts of >= 256 columns
    hp.wq = round_up((n + hp.q - 1) / hp.q, 128);  // even column offsets keep C blocks 16-B aligned
    hp.q = int((n + hp.wq - 1) / hp.wq);
    // front parts in eighths of q (tuning: TCEC_HOST_BFRONT).  A quarter of B
    // ahead of A: the GEMM (not the H2D) bounds the TF32TCEC headline, so a
    // shorter head wins (16384^3 on the reference inputs: e2e 207.6 / 216.4 /
    // 218.0 TFLOP/s with 4 / 3 / 2 eighths, 0 reruns; profiles/r02_host_bfront_ab.log).
    // The decision taken from fewer parts is checked against the exact one
    // (rerun on disagreement), so only speed depends on it.
    static const int front_num = [] {
        const char* e = std::getenv("TCEC_HOST_BFRONT");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 && v <= 8 ? v : 2;
    }();
    hp.front = std::max(1, hp.q * front_num / 8);
    return hp;
}

// Host<->device copies of the host-buffer entry point: direct DMA for pinned
// buffers, the pinned staging ring (host_stage.h) for pageable ones.
struct HostIO {
    bool a_dma = true, b_dma = true, c_dma = true;
    StageRing* ring = nullptr;
    cudaError_t h2d(bool dma_ok, uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width,
                    size_t height, cudaStream_t st) const {
        if (dma_ok)
            return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, st);
        if (height == 1 && width > StageRing::kSlotBytes) {  // one flat buffer: slot-sized pieces
            for (size_t off = 0; off < width; off += StageRing::kSlotBytes) {
                const size_t w = std::min(StageRing::kSlotBytes, width - off);
                const cudaError_t e = ring->h2d(dst + off, w, src + off, w, w, 1, st);
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        }
        return ring->h2d(dst, dpitch, src, spitch, width, height, st);
    }
    cudaError_t d2h(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width,
                    size_t height, cudaStream_t st) const {
        if (c_dma)
            return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, st);
        return ring->d2h(dst, dpitch, src, spitch, width, height, st);
    }
};

static int host_pipeline(Handle& h, const uint8_t* a, const uint8_t* b, uint8_t* c, int64_t m,
                         int64_t n, int64_t k, const tcec_dispatch_config_t& cfg,
                         const DispatchPlan& p, void* ws, uint8_t* da, uint8_t* db, uint8_t* dc,
                         const HostPipe& hp, DevDecision* d, const HostIO& io) {
    cudaStream_t s = h.stream;
    if (!h.in_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h.in_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&h.gemm_stream2, cudaStreamNonBlocking));
        for (auto& e : h.in_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    DevDecision* dr = d;        // exact decision (all of A and B)
    DevDecision* ds = d + 1;    // decision the blocks run under
    DevDecision* snap = d + 2;  // ds right after selection (before prep adds its flags)
    const size_t row_bytes = size_t(k) * 8;
    auto j0_of = [&](int j) { return int64_t(j) * hp.wq; };
    auto w_of = [&](int j) { return std::min(hp.wq, n - j0_of(j)); };
    cudaEvent_t* ev_b = h.in_ev;              // B column parts
    cudaEvent_t* ev_a = h.in_ev + hp.q;       // A row chunks
    cudaEvent_t ev_sync = h.in_ev[40];        // stream-to-stream ordering
    // the staging buffers may still be read by earlier work on the stream
    CUDA_TRY(cudaEventRecord(ev_sync, s));
    CUDA_TRY(cudaStreamWaitEvent(h.in_stream, ev_sync, 0));
    auto put_b = [&](int j) -> int {
        const int64_t j0 = j0_of(j), w = w_of(j);
        CUDA_TRY(io.h2d(io.b_dma, db + size_t(k) * j0 * 8, size_t(w) * 8, b + j0 * 8, size_t(n) * 8,
                        size_t(w) * 8, size_t(k), h.in_stream));
        CUDA_TRY(cudaEventRecord(ev_b[j], h.in_stream));
        return TCEC_OK;
    };
    for (int j = 0; j < hp.front; ++j)
        if (int rc = put_b(j)) return rc;
    for (int i = 0; i < hp.nch; ++i) {
        const int64_t r0 = i * hp.rows_per, r1 = std::min(m, r0 + hp.rows_per);
        CUDA_TRY(io.h2d(io.a_dma, da + r0 * row_bytes, row_bytes, a + r0 * row_bytes, row_bytes, row_bytes,
                        size_t(r1 - r0), h.in_stream));
        CUDA_TRY(cudaEventRecord(ev_a[i], h.in_stream));
    }
    for (int j = hp.front; j < hp.q; ++j)
        if (int rc = put_b(j)) return rc;

    const float* fa = reinterpret_cast<const float*>(da);
    const float* fb = reinterpret_cast<const float*>(db);
    for (int j = 0; j < hp.front; ++j) CUDA_TRY(cudaStreamWaitEvent(s, ev_b[j], 0));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_a[0], 0));
    cudaMemsetAsync(ds, 0, sizeof(DevDecision), s);
    const double t = p.forced_scaled ? 1.0 : cfg.threshold_t;
    const int64_t rows0 = std::min(m, hp.rows_per);
    const int64_t bfront = k * std::min(n, j0_of(hp.front));  // the packed front parts
    if (p.stats) {
        launch_stats1(fa, 2 * rows0 * k, fb, 2 * bfront, ds, s);
        const float fa_frac = host_spec_tf32() ? float(double(rows0) / double(m)) : 0.0f;
        const float fb_frac = host_spec_tf32() ? float(double(bfront) / double(k * n)) : 0.0f;
        launch_stats2(fa, 2 * rows0 * k, fb, 2 * bfront, ds, t, cfg.target_max_exponent, 0, s, 1,
                      cfg.threshold_t, p.forced_scaled ? 1 : 0, fa_frac, fb_frac);
        cudaMemcpyAsync(snap, ds, sizeof(DevDecision), cudaMemcpyDeviceToDevice, s);
    }
    TcecGemmArgs g = tc_gemm_args(h, p, ws, reinterpret_cast<float*>(dc), m, n, ds, false);
    g.ldc = 2 * n;
    g.no_split = 1;
    void* bhi = const_cast<void*>(g.b_hi);
    void* blo = const_cast<void*>(g.b_lo);
    auto prep_part = [&](int j) {
        launch_prep_b(fb + 2 * k * j0_of(j), k, w_of(j), p.kp, bhi, blo, ds, p.kind, p.corrected, s,
                      j0_of(j));
    };
    int unit = 0;
    // GEMM of rows [r0, r1) x columns [c0, c0 + w), then its block of C goes back
    auto block = [&](int64_t r0, int64_t r1, int64_t c0, int64_t w) -> int {
        cudaStream_t gs = (unit++ & 1) ? h.gemm_stream2 : s;
        if (gs != s) {
            CUDA_TRY(cudaEventRecord(ev_sync, s));  // the preps this block reads
            CUDA_TRY(cudaStreamWaitEvent(gs, ev_sync, 0));
        }
        TcecGemmArgs gb = g;
        gb.m = r1 - r0;
        gb.a_row_off = r0;
        gb.n2 = 2 * w;
        gb.b_row_off = 2 * c0;
        gb.c = g.c + r0 * 2 * n + 2 * c0;
        const int e = launch_tcec_gemm(gb, gs);
        if (e) return cuda_error(cudaError_t(e), "tcec_gemm (host pipeline)");
        cudaEvent_t ev = h.chunk_ev[unit % 8];
        CUDA_TRY(cudaEventRecord(ev, gs));
        CUDA_TRY(cudaStreamWaitEvent(h.copy_stream, ev, 0));
        const size_t off = size_t(r0 * n + c0) * 8;
        CUDA_TRY(io.d2h(c + off, size_t(n) * 8, dc + off, size_t(n) * 8, size_t(w) * 8, size_t(r1 - r0),
                        h.copy_stream));
        return TCEC_OK;
    };
    for (int j = 0; j < hp.front; ++j) prep_part(j);
    const int64_t wfront = std::min(n, j0_of(hp.front));  // front parts are contiguous columns
    for (int i = 0; i < hp.nch; ++i) {
        const int64_t r0 = i * hp.rows_per, r1 = std::min(m, r0 + hp.rows_per);
        CUDA_TRY(cudaStreamWaitEvent(s, ev_a[i], 0));
        launch_prep_a(fa, r1 - r0, k, p.kp, const_cast<void*>(g.a_hi), const_cast<void*>(g.a_lo), ds,
                      p.kind, p.corrected, s, r0);
        if (int rc = block(r0, r1, 0, wfront)) return rc;
    }
    for (int j = hp.front; j < hp.q; ++j) {
        CUDA_TRY(cudaStreamWaitEvent(s, ev_b[j], 0));
        prep_part(j);
        for (int i = 0; i < hp.nch; ++i) {
            const int64_t r0 = i * hp.rows_per, r1 = std::min(m, r0 + hp.rows_per);
            if (int rc = block(r0, r1, j0_of(j), w_of(j))) return rc;
        }
    }
    if (p.stats) {
        cudaMemsetAsync(dr, 0, sizeof(DevDecision), s);
        launch_stats1(fa, 2 * m * k, fb, 2 * k * n, dr, s);
        launch_stats2(fa, 2 * m * k, fb, 2 * k * n, dr, t, cfg.target_max_exponent, 0, s, 1, cfg.threshold_t,
                      p.forced_scaled ? 1 : 0);
    }
    CUDA_TRY(cudaEventRecord(ev_sync, h.gemm_stream2));  // s covers the second GEMM stream
    CUDA_TRY(cudaStreamWaitEvent(s, ev_sync, 0));
    CUDA_TRY(cudaGetLastError());
    return TCEC_OK;
}

int tcec_dispatch_cgemm_host(tcec_handle h, const void* a, const void* b, void* c, int64_t m,
                             int64_t n, int64_t k, const tcec_dispatch_config_t* cfg,
                             tcec_dispatch_result_t* res) {
    CHECK_HANDLE(h);
    if (!cfg || !res) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (m < 0 || n < 0 || k < 0) return set_error(TCEC_ERR_SHAPE_MISMATCH, "negative extent");
    const size_t ab = size_t(m) * k * 8, bb = size_t(k) * n * 8, cb = size_t(m) * n * 8;
    const size_t ra = size_t(round_up(int64_t(ab), 256)), rb = size_t(round_up(int64_t(bb), 256));
    const size_t need = ra + rb + cb + 256;
    if (h->io_bytes < need) {
        cudaStreamSynchronize(h->stream);
        if (h->io) cudaFree(h->io);
        h->io = nullptr;
        h->io_bytes = 0;
        CUDA_TRY(cudaMalloc(&h->io, need));
        h->io_bytes = need;
    }
    uint8_t* base = static_cast<uint8_t*>(h->io);
    uint8_t* da = base;
    uint8_t* db = base + ra;
    uint8_t* dc = base + ra + rb;
    // the GEMM runs in row chunks; each finished chunk of C is copied back on
    // a second stream while the next chunk computes
    if (!h->copy_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        for (auto& e : h->chunk_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const DispatchPlan p = plan_dispatch(m, n, k, *cfg);
    void* ws = nullptr;
    const size_t wsb = plan_workspace(p, m, n);
    if (wsb) {
        ws = h->workspace(wsb);
        if (!ws) return set_error(TCEC_ERR_CUDA, "workspace allocation failed");
    }
    // pageable host buffers (a std::vector, a numpy array) go through the
    // pinned staging ring so the copies stay asynchronous and overlapped
    HostIO io;
    io.a_dma = ab == 0 || dma_capable(a);
    io.b_dma = bb == 0 || dma_capable(b);
    io.c_dma = cb == 0 || dma_capable(c);
    if (!(io.a_dma && io.b_dma && io.c_dma)) {
        if (!h->stage) h->stage = std::make_unique<StageRing>();
        CUDA_TRY(h->stage->init());
        io.ring = h->stage.get();
    }
    auto finish_io = [&]() -> int {
        if (io.ring) {
            CUDA_TRY(cudaStreamSynchronize(io.ring->host));
            io.ring->finish();
        }
        return TCEC_OK;
    };
    struct Ctx {
        tcec_handle h;
        uint8_t* c_host;
        const uint8_t* dc;
        int64_t row_bytes;
        int used;
        cudaError_t err;
        const HostIO* io;
    } ctx{h, static_cast<uint8_t*>(c), dc, n * 8, 0, cudaSuccess, &io};
    ChunkHook hook;
    hook.chunks = m >= 8192 ? 4 : 1;
    hook.ctx = &ctx;
    hook.done = [](void* vp, int64_t r0, int64_t r1) -> int {
        Ctx& x = *static_cast<Ctx*>(vp);
        cudaEvent_t ev = x.h->chunk_ev[x.used++ % 8];
        cudaError_t e = cudaEventRecord(ev, x.h->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(x.h->copy_stream, ev, 0);
        if (e == cudaSuccess)
            e = x.io->d2h(x.c_host + r0 * x.row_bytes, size_t(x.row_bytes), x.dc + r0 * x.row_bytes,
                          size_t(x.row_bytes), size_t(x.row_bytes), size_t(r1 - r0), x.h->copy_stream);
        if (e != cudaSuccess) {
            x.err = e;
            return cuda_error(e, "chunk copy");
        }
        return TCEC_OK;
    };
    // operand copies overlapped with the GEMM (host_pipeline) for large
    // tensor-core dispatches; TCEC_HOST_CHUNKS = 0 disables.  16 row chunks of
    // A (1024 rows at 16384^3): e2e / device 0.945-0.950 against 0.919-0.922
    // with 12 and 0.906-0.931 with 24-32 (profiles/r02e_host_chunks_sweep.log)
    static const int pipe_chunks = [] {
        const char* e = std::getenv("TCEC_HOST_CHUNKS");
        return e ? std::max(0, std::min(32, std::atoi(e))) : 16;
    }();
    static const int pipe_parts = [] {  // column parts of B (front half sent before A)
        const char* e = std::getenv("TCEC_HOST_BPARTS");
        return e ? std::max(1, std::min(8, std::atoi(e))) : 8;
    }();
    const bool pipelined = pipe_chunks > 1 && p.tier == kTierTc && m >= 8192 && n > 0 && k > 0 &&
                           !(h->prof && h->ev[0]) &&
                           (resolve_gemm_variant(h->gemm_pair, m, 2 * n, p.kp, h->sm_count, false, false) ==
                                kVariantWide ||
                            resolve_gemm_variant(h->gemm_pair, m, 2 * n, p.kp, h->sm_count, false, false) ==
                                kVariantWideMc);
    DevDecision* d = pipelined ? h->decisions(3) : h->dec;
    if (!d) return set_error(TCEC_ERR_CUDA, "decision slots allocation failed");
    if (pipelined) {
        const HostPipe hp = plan_host_pipe(m, n, pipe_chunks, pipe_parts);
        int rc = host_pipeline(*h, static_cast<const uint8_t*>(a), static_cast<const uint8_t*>(b),
                               static_cast<uint8_t*>(c), m, n, k, *cfg, p, ws, da, db, dc, hp, d, io);
        if (rc) return rc;
        ++h->pipe_runs;
        CUDA_TRY(cudaMemcpyAsync(h->dec_host, d, 3 * sizeof(DevDecision), cudaMemcpyDeviceToHost,
                                 h->stream));
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        CUDA_TRY(cudaStreamSynchronize(h->copy_stream));
        if ((rc = finish_io())) return rc;
        const DevDecision& dr = h->dec_host[0];
        const DevDecision& ds = h->dec_host[1];
        const DevDecision& snap = h->dec_host[2];
        if (!p.stats) return finish_dispatch(p, ds, m, n, k, res);
        if (dr.kind == snap.kind && dr.scale_a == snap.scale_a && dr.scale_b == snap.scale_b &&
            dr.overflow == snap.overflow && dr.scale_overflow == snap.scale_overflow) {
            DevDecision merged = dr;
            merged.overflow = ds.overflow;
            merged.scale_overflow = ds.scale_overflow;
            return finish_dispatch(p, merged, m, n, k, res);
        }
        if (std::getenv("TCEC_DEBUG_RERUN"))
            std::fprintf(stderr,
                         "rerun: exact kind %d sa %d sb %d ovf %u sovf %u (e_max %d/%d n1 %llu/%llu nz %llu/%llu n2 %llu/%llu) | "
                         "spec kind %d sa %d sb %d ovf %u sovf %u (e_max %d/%d n1 %llu/%llu nz %llu/%llu n2 %llu/%llu)\n",
                         dr.kind, dr.scale_a, dr.scale_b, dr.overflow, dr.scale_overflow, dr.st[0].e_max,
                         dr.st[1].e_max, dr.st[0].n1, dr.st[1].n1, dr.st[0].n_nonzero, dr.st[1].n_nonzero,
                         dr.st[0].n2, dr.st[1].n2, snap.kind, snap.scale_a, snap.scale_b, snap.overflow,
                         snap.scale_overflow, snap.st[0].e_max, snap.st[1].e_max, snap.st[0].n1, snap.st[1].n1,
                         snap.st[0].n_nonzero, snap.st[1].n_nonzero, snap.st[0].n2, snap.st[1].n2);
        // the first chunks were not representative: plain path on the resident A
        // and a row-major copy of B (the staging holds it packed by column part)
        ctx.used = 0;
        ++h->pipe_reruns;
        CUDA_TRY(io.h2d(io.b_dma, db, bb, static_cast<const uint8_t*>(b), bb, bb, bb ? 1 : 0, h->stream));
    } else {
        CUDA_TRY(io.h2d(io.a_dma, da, ab, static_cast<const uint8_t*>(a), ab, ab, ab ? 1 : 0, h->stream));
        CUDA_TRY(io.h2d(io.b_dma, db, bb, static_cast<const uint8_t*>(b), bb, bb, bb ? 1 : 0, h->stream));
    }
    int rc = launch_dispatch(*h, reinterpret_cast<const float*>(da), reinterpret_cast<const float*>(db),
                             reinterpret_cast<float*>(dc), m, n, k, *cfg, p, d, ws, &hook);
    if (rc) return rc;
    CUDA_TRY(cudaGetLastError());
    if (ctx.used == 0 && m > 0 && n > 0)
        CUDA_TRY(io.d2h(static_cast<uint8_t*>(c), size_t(n) * 8, dc, size_t(n) * 8, size_t(n) * 8, size_t(m),
                        h->stream));
    CUDA_TRY(cudaMemcpyAsync(h->dec_host, d, sizeof(DevDecision), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->copy_stream));
    if (int rc = finish_io()) return rc;
    if (h->prof && h->ev[0]) {
        for (int i = 0; i < 3; ++i) {
            float ms = 0.0f;
            if (cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]) == cudaSuccess) h->prof_ms[i] += ms;
        }
        ++h->prof_count;
    }
    return finish_dispatch(p, *h->dec_host, m, n, k, res);
}

// ---------------------------------------------------------------- permute

int tcec_permute(tcec_handle h, const void* src, void* dst, int rank, const int64_t* old_dims,
                 const int* axis_of) {
    CHECK_HANDLE(h);
    if (rank < 0 || rank > kMaxRank)
        return set_error(TCEC_ERR_INVALID_PERMUTATION, "permutation has wrong length");
    bool used[kMaxRank] = {false};
    for (int a = 0; a < rank; ++a) {
        const int o = axis_of[a];
        if (o < 0 || o >= rank || used[o])
            return set_error(TCEC_ERR_INVALID_PERMUTATION, "label not in tensor: axis " +
                                                               std::to_string(o));
        used[o] = true;
        if (old_dims[a] < 1) return set_error(TCEC_ERR_SHAPE_MISMATCH, "tensor extents must be >= 1");
    }
    if (rank == 0) {
        CUDA_TRY(cudaMemcpyAsync(dst, src, 8, cudaMemcpyDeviceToDevice, h->stream));
        return TCEC_OK;
    }
    launch_permute(static_cast<const float2*>(src), static_cast<float2*>(dst), rank, old_dims,
                   axis_of, h->stream);
    CUDA_TRY(cudaGetLastError());
    return TCEC_OK;
}

}  // extern "C"
