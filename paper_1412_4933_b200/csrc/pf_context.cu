// C-ABI of pedflow-b200 (include/pf_gpu.h): context lifetime, state
// upload/download, the step loop (CUDA-graph batched), halo support.
#include "../../include/pf_gpu.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "pf_internal.h"
#include "pf_setup.h"

using pfdev::kWall;

namespace {

thread_local std::string g_err;

// NVTX ranges around every C-ABI entry point that does device work (SURVEY
// §5 tracing): visible in Nsight Systems / ncu --nvtx as pf_step,
// pf_load_state, ... (header-only NVTX3: no cost without an attached tool).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define PF_CUDA(call)                                                                             \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return fail(PF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Run fn(begin, end) over [0, n) on the host's threads (state conversion),
// on the library's persistent worker pool.
static void host_parallel(size_t n, const std::function<void(size_t, size_t)>& fn) {
    pfhost::pool_for(n, std::min<size_t>(2 * (pfhost::pool_threads() + 1), std::max<size_t>(1, n / 64)), fn);
}

// Large host<->device copies of the caller's pageable planes. A plain
// cudaMemcpy from pageable memory is staged by the driver through a small
// pinned buffer with one host thread (a few GB/s). Here the host side of each
// chunk is a multi-threaded memcpy into / out of our own pinned double buffer
// and the DMA of chunk i overlaps the host copy of chunk i-1 (or i+1).
class Stager {
  public:
    static constexpr size_t kChunk = size_t(64) << 20;
    static constexpr size_t kDirect = size_t(4) << 20;  // smaller copies go direct

    ~Stager() {
        for (int i = 0; i < 2; ++i) {
            if (ev_[i]) cudaEventDestroy(ev_[i]);
            if (buf_[i]) cudaFreeHost(buf_[i]);
        }
    }

    // Page-locked caller memory (pf_host_alloc, cudaHostAlloc/Register) is
    // DMA'd directly; pageable memory goes through the staging buffers.
    static bool pinned(const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }

    cudaError_t h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
        if (n < kDirect || pinned(src)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s);
        if (cudaError_t e = ready()) return e;
        const size_t nch = (n + kChunk - 1) / kChunk;
        for (size_t i = 0; i < nch; ++i) {
            const int slot = int(i & 1);
            const size_t off = i * kChunk, len = std::min(kChunk, n - off);
            if (cudaError_t e = cudaEventSynchronize(ev_[slot])) return e;  // DMA of chunk i-2 done
            par_copy(buf_[slot], static_cast<const char*>(src) + off, len);
            if (cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[slot], len, cudaMemcpyHostToDevice, s))
                return e;
            if (cudaError_t e = cudaEventRecord(ev_[slot], s)) return e;
        }
        return cudaSuccess;
    }

    cudaError_t d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
        if (n < kDirect || pinned(dst)) {
            cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s);
            return e ? e : cudaStreamSynchronize(s);
        }
        if (cudaError_t e = ready()) return e;
        const size_t nch = (n + kChunk - 1) / kChunk;
        for (size_t i = 0; i <= nch; ++i) {
            if (i < nch) {
                const int slot = int(i & 1);
                const size_t off = i * kChunk, len = std::min(kChunk, n - off);
                if (cudaError_t e = cudaMemcpyAsync(buf_[slot], static_cast<const char*>(src) + off, len,
                                                    cudaMemcpyDeviceToHost, s))
                    return e;
                if (cudaError_t e = cudaEventRecord(ev_[slot], s)) return e;
            }
            if (i >= 1) {
                const size_t j = i - 1, off = j * kChunk, len = std::min(kChunk, n - off);
                if (cudaError_t e = cudaEventSynchronize(ev_[j & 1])) return e;
                par_copy(static_cast<char*>(dst) + off, buf_[j & 1], len);
            }
        }
        return cudaSuccess;
    }

    // Allocate the pinned buffers now (pf_create does this for large grids so
    // that the first state transfer does not pay for it).
    cudaError_t ready() {
        for (int i = 0; i < 2; ++i) {
            if (!ev_[i])
                if (cudaError_t e = cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming)) return e;
            if (!buf_[i])
                if (cudaError_t e = cudaHostAlloc(&buf_[i], kChunk, cudaHostAllocDefault)) return e;
        }
        return cudaSuccess;
    }

  private:
    // Host side of a chunk: a memcpy split over the library's persistent
    // worker pool (spawning threads per 64 MB chunk cost a third of the
    // transfer time at C5).
    static void par_copy(void* dst, const void* src, size_t n) {
        const size_t pages = (n + 4095) / 4096;
        pfhost::pool_for(pages, std::min<size_t>(pages, 2 * (pfhost::pool_threads() + 1)), [&](size_t b0, size_t b1) {
            const size_t lo = std::min(n, b0 * 4096), hi = std::min(n, b1 * 4096);
            if (hi > lo) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
        });
    }
    void* buf_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
};

// PEDFLOW_IO_TRACE=1: per-phase wall times of state load/store on stderr (dev).
struct IoTrace {
    bool on = std::getenv("PEDFLOW_IO_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void operator()(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[pedflow io] %-48s %8.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

constexpr int kBatchCap = 256;   // steps per captured CUDA graph
constexpr int kReportCap = 1024; // report ring slots per replica (slot = step % kReportCap)

}  // namespace

struct pf_ctx {
    pf_config cfg{};
    pfk::StepArgs args{};
    int rows_owned = 0, rows_buf = 0, row_begin = 0;
    int parity = 0;                 // buffer holding the current state
    uint32_t step = 0;              // host mirror of the device step counter
    uint32_t* d_step = nullptr;
    uint32_t* d_reports = nullptr;  // [replicas][kReportCap][4] ring
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;  // side stream for host<->device state transfers
    uint64_t launches = 0;
    std::map<std::pair<uint32_t, int>, cudaGraphExec_t> graphs;
    std::map<std::pair<uint32_t, int>, uint64_t> graph_launches;  // kernel launches per replay
    std::vector<void*> allocs;
    Stager stage[2];                            // [0] main thread, [1] side thread
    void* io_scratch = nullptr;                 // device staging of exported SimState planes
    size_t io_scratch_bytes = 0;
    cudaEvent_t io_event = nullptr;
    // Fused halo exchange: d_sync[side] = steps completed by the linked
    // neighbour on that side (written by it); remote_flag[side] = the
    // neighbour's flag for us; d_err = handshake timeout.
    uint32_t* d_sync = nullptr;
    uint32_t* d_err = nullptr;
    uint32_t* remote_flag[2] = {nullptr, nullptr};
    int linked = 0;                             // bit s: neighbour on side s
    bool multistep = true;                      // PF_KERNEL_FUSED, unlinked: one launch per batch of steps
    size_t tile_done_bytes = 0;
    std::vector<void*> ipc_opened;              // peer allocations opened with cudaIpcOpenMemHandle
    // Phase-level stepping (pf_phase, PF_KERNEL_PIPELINE): 0 between steps,
    // else the last phase done + 1; CandidateScores by agent id.
    int phase = 0;
    double* d_scores = nullptr;
    uint32_t scores_n = 0;                      // agents per replica slot of d_scores
    std::vector<int32_t> rep_aps;               // agents_per_side of each replica
    std::vector<pfdev::ReplicaParams> reps;     // host copy of args.rep
    bool aco() const { return cfg.model == PF_MODEL_ACO; }
    bool bits() const { return cfg.kernel == PF_KERNEL_FUSED || cfg.kernel == PF_KERNEL_FUSED_F32; }  // occupancy planes + in-place words
    bool f32() const { return cfg.kernel == PF_KERNEL_FUSED_F32 && aco(); }  // pheromone stored as float2
    size_t tau_elem() const { return f32() ? 8 : 16; }
    // Element `elem` of pheromone buffer `buf` (double2 or float2 storage).
    void* tau_ptr(int buf, size_t elem) const { return reinterpret_cast<char*>(args.p.tau[buf]) + elem * tau_elem(); }
    size_t plane() const { return size_t(rows_buf) * size_t(cfg.width); }
    size_t total() const { return plane() * size_t(cfg.replicas); }
};

extern "C" {

const char* pf_last_error(void) { return g_err.c_str(); }
const char* pf_version(void) { return "pedflow-b200 0.1 (sm_100a)"; }

int32_t pf_band_height(int32_t n, int32_t w) { return pfhost::band_height(n, w); }

int pf_validate(const pf_config* c) {
    if (!c) return fail(PF_ERR_ARG, "null config");
    // validate() (src/config.cpp:101-124)
    if (c->width < 16 || c->width % 16 != 0) return fail(PF_ERR_CONFIG, "width must be a multiple of 16 and >= 16");
    if (c->height < 16 || c->height % 16 != 0) return fail(PF_ERR_CONFIG, "height must be a multiple of 16 and >= 16");
    if (c->agents_per_side < 0) return fail(PF_ERR_CONFIG, "agents_per_side must be >= 0");
    if (c->model != PF_MODEL_LEM && c->model != PF_MODEL_ACO) return fail(PF_ERR_CONFIG, "malformed value for key 'model'");
    if (!(c->d0 > 1.0)) return fail(PF_ERR_CONFIG, "d0 must be > 1");
    if (!(c->sel_sigma >= 0.0)) return fail(PF_ERR_CONFIG, "sel_sigma must be >= 0");
    if (!(c->alpha >= 0.0)) return fail(PF_ERR_CONFIG, "alpha must be >= 0");
    if (!(c->beta >= 0.0)) return fail(PF_ERR_CONFIG, "beta must be >= 0");
    if (!(c->rho > 0.0 && c->rho <= 1.0)) return fail(PF_ERR_CONFIG, "rho must be in (0, 1]");
    if (!(c->tau0 > 0.0)) return fail(PF_ERR_CONFIG, "tau0 must be > 0");
    if (!(c->q > 0.0)) return fail(PF_ERR_CONFIG, "q must be > 0");
    const int64_t cells = int64_t(c->width) * c->height;
    if (2 * int64_t(c->agents_per_side) > cells)
        return fail(PF_ERR_CONFIG, "agents_per_side exceeds grid capacity (width * height / 2)");
    const int band = pfhost::band_height(c->agents_per_side, c->width);
    if (2 * band > c->height)
        return fail(PF_ERR_CONFIG, "agents_per_side needs more placement rows than the grid height allows");
    // GPU preconditions
    if (cells >= (int64_t(1) << 32)) return fail(PF_ERR_CONFIG, "width * height must be < 2^32");
    if (2 * int64_t(c->agents_per_side) >= (int64_t(1) << 29)) return fail(PF_ERR_CONFIG, "2 * agents_per_side must be < 2^29");
    if (c->replicas < 1) return fail(PF_ERR_CONFIG, "replicas must be >= 1");
    if (c->replicas > 65535) return fail(PF_ERR_CONFIG, "replicas must be <= 65535");
    if (c->kernel != PF_KERNEL_FUSED && c->kernel != PF_KERNEL_PIPELINE && c->kernel != PF_KERNEL_TILE &&
        c->kernel != PF_KERNEL_FUSED_F32)
        return fail(PF_ERR_CONFIG, "unknown kernel");
    if (c->row_end != 0) {
        if (c->row_begin < 0 || c->row_end > c->height || c->row_begin >= c->row_end)
            return fail(PF_ERR_CONFIG, "shard rows must satisfy 0 <= row_begin < row_end <= height");
        if (c->row_end - c->row_begin < PF_GHOST_ROWS)
            return fail(PF_ERR_CONFIG, "a row shard must own at least PF_GHOST_ROWS rows");
    }
    return PF_OK;
}

int pf_new_environment(const pf_config* c, uint64_t seed, uint8_t* occ, uint32_t* index, pf_agent* agents,
                       double* tau_top, double* tau_bot) {
    pf_config v = *c;
    v.replicas = 1;
    v.row_begin = v.row_end = 0;
    if (int rc = pf_validate(&v)) return rc;
    if (!occ || !index || (!agents && c->agents_per_side > 0)) return fail(PF_ERR_ARG, "null plane");
    const size_t cells = size_t(c->width) * size_t(c->height);
    const size_t n_agents = c->agents_per_side > 0 ? 2 * size_t(c->agents_per_side) : 0;
    const bool tau = c->model == PF_MODEL_ACO && tau_top && tau_bot;
    pfhost::parallel_for(cells, [&](size_t b, size_t e) {  // host-memory bound: all cores (C5: 7.4 GB)
        std::memset(occ + b, 0, e - b);
        std::memset(index + b, 0, (e - b) * 4);
        if (tau) {
            std::fill(tau_top + b, tau_top + e, c->tau0);
            std::fill(tau_bot + b, tau_bot + e, c->tau0);
        }
    });
    pfhost::parallel_for(n_agents, [&](size_t b, size_t e) { std::memset(agents + b, 0, sizeof(pf_agent) * (e - b)); });
    const uint32_t W = uint32_t(c->width);
    try {
    pfhost::place_all(c->width, c->height, c->agents_per_side, seed, [&](uint32_t cell, uint32_t id, uint32_t g) {
        occ[cell] = uint8_t(g);
        index[cell] = id;
        pf_agent& a = agents[id - 1];
        a.index = id;
        a.group = uint8_t(g);
        a.row = a.future_row = int32_t(cell / W);
        a.col = a.future_col = int32_t(cell % W);
        a.tour_length = 0.0;
        a.crossed = 0;
    });
    } catch (const std::exception& e) {
        return fail(PF_ERR_ARG, std::string("new_environment: ") + e.what());
    }
    return PF_OK;
}

int pf_destroy(pf_ctx* ctx) {
    if (!ctx) return PF_OK;
    cudaSetDevice(ctx->cfg.device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    for (void* p : ctx->allocs) cudaFree(p);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
    if (ctx->io_scratch) cudaFree(ctx->io_scratch);
    if (ctx->io_event) cudaEventDestroy(ctx->io_event);
    if (ctx->d_scores) cudaFree(ctx->d_scores);
    delete ctx;
    return PF_OK;
}

// StepArgs::skip_empty: the widest replica's two starting bands cover under
// 30% of the grid's rows.
static void set_skip_empty(pf_ctx* ctx) {
    int band = 0;
    for (const auto& r : ctx->reps) band = std::max(band, int(r.band));
    ctx->args.skip_empty = 2.0 * band < 0.3 * ctx->cfg.height ? 1 : 0;
}

// Small sparse LEM grids run on the cluster-resident kernel (pf_cluster.cu).
static void set_cluster(pf_ctx* ctx) {
    uint32_t most = 0;
    for (const auto& r : ctx->reps) most = std::max(most, r.n_agents);
    ctx->args.cluster_cap = 0;
    ctx->args.cluster_nt = 1024;
    ctx->args.cluster =
        ctx->bits() ? pfk::plan_cluster_lem(ctx->args, most, &ctx->args.cluster_cap, &ctx->args.cluster_nt) : 0;
}

static int fill_consts(pf_ctx* ctx) {
    const pf_config& c = ctx->cfg;
    pfdev::StepConsts& k = ctx->args.k;
    // distance_table (src/grid.cpp:10-27) and the host-side factors the
    // reference computes once: dmin/d_i (src/lem.cpp:11-16), (1/d_i)^beta
    // (src/aco.cpp:24), 1 - rho (src/engine.cpp:126), sqrt(2) (src/aco.cpp:11).
    const int f[8] = {+1, +1, +1, 0, 0, -1, -1, -1};
    const int l[8] = {0, 1, 1, 1, 1, 0, 1, 1};
    double d[8];
    for (int i = 0; i < 8; ++i) d[i] = std::sqrt((c.d0 - f[i]) * (c.d0 - f[i]) + double(l[i] * l[i]));
    for (int i = 0; i < 8; ++i) {
        k.lem_score[i] = d[0] / d[i];
        k.eta[i] = std::pow(1.0 / d[i], c.beta);
    }
    // The device's lem_select takes C_max as the first open slot's score:
    // scores must not grow with the slot index (true for every d0 > 1).
    for (int i = 1; i < 8; ++i)
        if (k.lem_score[i] > k.lem_score[i - 1]) return fail(PF_ERR_CONFIG, "distance table not monotone in slot order");
    k.sel_mu = c.sel_mu;
    k.sel_sigma = c.sel_sigma;
    k.alpha = c.alpha;
    k.alpha_mode = c.alpha == 1.0 ? 0 : (c.alpha == 0.0 ? 1 : 2);
    k.factor = 1.0 - c.rho;
    k.q = c.q;
    k.diag = std::sqrt(2.0);
    k.model = c.model;
    k.W = c.width;
    k.H = c.height;
    return PF_OK;
}

int pf_create(const pf_config* cfg, pf_ctx** out) {
    NvtxRange nvtx_range("pf_create");
    if (!out) return fail(PF_ERR_ARG, "null out");
    *out = nullptr;
    if (int rc = pf_validate(cfg)) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PF_ERR_CUDA, "no CUDA device available");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(PF_ERR_CONFIG, "device ordinal out of range");
    auto* ctx = new pf_ctx();
    ctx->cfg = *cfg;
    ctx->row_begin = cfg->row_end ? cfg->row_begin : 0;
    ctx->rows_owned = cfg->row_end ? cfg->row_end - cfg->row_begin : cfg->height;
    ctx->rows_buf = ctx->rows_owned + 2 * pfk::kGhost;
    auto cleanup = [&](int rc) {
        pf_destroy(ctx);
        return rc;
    };
    if (int rc = fill_consts(ctx)) return cleanup(rc);
    if (cudaSetDevice(cfg->device) != cudaSuccess) return cleanup(fail(PF_ERR_CUDA, "cudaSetDevice failed"));
    if (pfk::configure_step_bits() != 0) return cleanup(fail(PF_ERR_CUDA, "cannot configure the step kernel's shared memory"));
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(fail(PF_ERR_CUDA, "cudaStreamCreate failed"));
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
        ctx->allocs.push_back(p);
        return p;
    };
    const size_t n = ctx->total();
    pfk::Planes& P = ctx->args.p;
    P.plane = ctx->plane();
    P.cell[0] = static_cast<uint32_t*>(alloc(n * 4));
    P.cell[1] = ctx->bits() ? P.cell[0] : static_cast<uint32_t*>(alloc(n * 4));
    bool ok = P.cell[0] && P.cell[1];
    if (ctx->bits()) {
        // Plane pitch: every strip's window (NS + 4 segments from segment
        // strip * NS - 2) lies inside the row, and rows stay 16-byte aligned.
        const int ns = pfk::bits_strip_segments(cfg->width, cfg->model, ctx->f32());
        ctx->args.strip_segs = ns;
        const int strips = (cfg->width + 32 * ns - 1) / (32 * ns);
        P.wsp = strips * ns + 4;
        P.occ_plane = size_t(ctx->rows_buf) * size_t(P.wsp);
        for (int i = 0; i < 2; ++i) {
            P.occ[i] = static_cast<uint2*>(alloc(P.occ_plane * size_t(cfg->replicas) * 8));
            ok = ok && P.occ[i];
        }
    }
    if (ctx->aco()) {
        P.tau[0] = static_cast<double2*>(alloc(n * 16));
        P.tau[1] = static_cast<double2*>(alloc(n * 16));
        P.tour = static_cast<double*>(alloc(n * 8));
        ok = ok && P.tau[0] && P.tau[1] && P.tour;
    }
    if (cfg->kernel == PF_KERNEL_PIPELINE) {
        P.intent = static_cast<uint8_t*>(alloc(n));
        P.win = static_cast<uint8_t*>(alloc(n));
        ok = ok && P.intent && P.win;
    }
    ctx->d_step = static_cast<uint32_t*>(alloc(4));
    ctx->d_sync = static_cast<uint32_t*>(alloc(8));
    ctx->d_err = static_cast<uint32_t*>(alloc(4));
    if (ctx->bits()) {
        // Per-tile completion flags of multi-step launches, sized for the
        // smallest tile geometry (64-column strips, 8-row tiles).
        ctx->tile_done_bytes = 4 * (size_t(cfg->replicas) * size_t((cfg->width + 63) / 64) *
                                        size_t((ctx->rows_owned + 7) / 8) + 1);
        ctx->args.tile_done = static_cast<uint32_t*>(alloc(ctx->tile_done_bytes));
        ok = ok && ctx->args.tile_done;
        const char* ms = std::getenv("PEDFLOW_MULTISTEP");  // dev: 0 = one launch per step
        ctx->multistep = !(ms && std::atoi(ms) == 0);
    }
    ctx->args.nsteps = 1;
    ctx->args.tau_f32 = ctx->f32() ? 1 : 0;
    ctx->args.bcount = static_cast<uint32_t*>(alloc(size_t(kReportCap) * 8));
    ok = ok && ctx->d_sync && ctx->d_err && ctx->args.bcount;
    ctx->args.sync_local = ctx->d_sync;
    ctx->args.err = ctx->d_err;
    auto* kc = static_cast<pfdev::StepConsts*>(alloc(sizeof(pfdev::StepConsts)));
    ok = ok && kc && cudaMemcpy(kc, &ctx->args.k, sizeof(pfdev::StepConsts), cudaMemcpyHostToDevice) == cudaSuccess;
    ctx->args.kc = kc;
    ctx->d_reports = static_cast<uint32_t*>(alloc(size_t(cfg->replicas) * kReportCap * 16));
    ctx->args.work = static_cast<uint32_t*>(alloc(size_t(kReportCap) * 4));
    {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
        ctx->args.num_sms = sms > 0 ? sms : 148;
        const char* ipc = std::getenv("PEDFLOW_ITEMS_PER_CTA");  // tuning override (dev)
        // Short items keep the end-of-step tail small; longer ones save item
        // claims and reuse the staged halo rows of consecutive tiles. Sweeps on
        // the final kernel: C5 LEM (32-row tiles) best at 16 items per CTA
        // (2 tiles per item); C5 ACO best with one tile per item (-1.2% against
        // 4), which 256 items per CTA gives for any grid up to ~110K tiles.
        ctx->args.items_per_cta = ipc ? std::max(1, std::atoi(ipc)) : (cfg->model == PF_MODEL_LEM ? 16 : 256);
        const char* st = std::getenv("PEDFLOW_SMALL_TILES");  // dev: force / forbid the small-grid geometry
        ctx->args.small_tiles = st ? (std::atoi(st) ? 1 : 0) : -1;
    }
    if (!ok || !ctx->d_step || !ctx->d_reports || !ctx->args.work) {
        cudaGetLastError();
        return cleanup(fail(PF_ERR_CUDA, "device allocation failed (out of memory?)"));
    }
    if (cudaMemsetAsync(P.cell[0], 0, n * 4, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(P.cell[1], 0, n * 4, ctx->stream) != cudaSuccess ||
        (P.occ[0] && cudaMemsetAsync(P.occ[0], 0xFF, P.occ_plane * size_t(cfg->replicas) * 8, ctx->stream) != cudaSuccess) ||
        (P.occ[1] && cudaMemsetAsync(P.occ[1], 0xFF, P.occ_plane * size_t(cfg->replicas) * 8, ctx->stream) != cudaSuccess) ||
        cudaMemsetAsync(ctx->d_step, 0, 4, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(ctx->d_sync, 0, 8, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(ctx->d_err, 0, 4, ctx->stream) != cudaSuccess ||
        (ctx->args.tile_done && cudaMemsetAsync(ctx->args.tile_done, 0, ctx->tile_done_bytes, ctx->stream) != cudaSuccess))
        return cleanup(fail(PF_ERR_CUDA, "cudaMemset failed"));
    if (P.intent) {
        ctx->launches += pfk::launch_fill_u8(P.intent, n, pfdev::kNone, ctx->stream);
        ctx->launches += pfk::launch_fill_u8(P.win, n, pfdev::kNone, ctx->stream);
    }
    ctx->rep_aps.assign(size_t(cfg->replicas), cfg->agents_per_side);
    ctx->reps.resize(size_t(cfg->replicas));
    for (int r = 0; r < cfg->replicas; ++r)
        ctx->reps[size_t(r)] = {cfg->seed + uint64_t(r), pfhost::band_height(cfg->agents_per_side, cfg->width),
                                2u * uint32_t(cfg->agents_per_side)};
    // Large grids: compute the placement (new_environment's keyed Fisher-Yates,
    // host work) in the background while the device is set up; the
    // pf_init_environment that normally follows finds it cached.
    if (size_t(cfg->width) * size_t(cfg->height) >= (size_t(1) << 20))
        for (int r = 0; r < std::min(cfg->replicas, 4); ++r)
            pfhost::prefetch_placement(cfg->width, cfg->height, cfg->agents_per_side, ctx->reps[size_t(r)].seed);
    set_skip_empty(ctx);
    {
        auto* d_rep = static_cast<pfdev::ReplicaParams*>(alloc(ctx->reps.size() * sizeof(pfdev::ReplicaParams)));
        if (!d_rep || cudaMemcpy(d_rep, ctx->reps.data(), ctx->reps.size() * sizeof(pfdev::ReplicaParams),
                                 cudaMemcpyHostToDevice) != cudaSuccess)
            return cleanup(fail(PF_ERR_CUDA, "device allocation failed (out of memory?)"));
        ctx->args.rep = d_rep;
    }
    ctx->args.d_step = ctx->d_step;
    ctx->args.reports = ctx->d_reports;
    ctx->args.report_cap = kReportCap;
    ctx->args.row_begin = ctx->row_begin;
    ctx->args.rows_owned = ctx->rows_owned;
    ctx->args.rows_buf = ctx->rows_buf;
    ctx->args.replicas = cfg->replicas;
    set_cluster(ctx);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return cleanup(fail(PF_ERR_CUDA, "init failed"));
    if (ctx->plane() * 4 >= Stager::kChunk &&
        (ctx->stage[0].ready() != cudaSuccess || ctx->stage[1].ready() != cudaSuccess))
        return cleanup(fail(PF_ERR_CUDA, "pinned staging allocation failed"));
    *out = ctx;
    return PF_OK;
}

int pf_set_replicas(pf_ctx* ctx, const int32_t* agents_per_side, const uint64_t* seeds) {
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    const int R = ctx->cfg.replicas;
    std::vector<pfdev::ReplicaParams> reps = ctx->reps;
    std::vector<int32_t> aps = ctx->rep_aps;
    for (int r = 0; r < R; ++r) {
        if (agents_per_side) {
            pf_config v = ctx->cfg;  // validate() of the replica's scenario (src/config.cpp:101-124)
            v.agents_per_side = agents_per_side[r];
            if (int rc = pf_validate(&v)) return rc;
            aps[size_t(r)] = v.agents_per_side;
            reps[size_t(r)].band = pfhost::band_height(v.agents_per_side, v.width);
            reps[size_t(r)].n_agents = 2u * uint32_t(v.agents_per_side);
        }
        if (seeds) reps[size_t(r)].seed = seeds[r];
    }
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    PF_CUDA(cudaMemcpy(const_cast<pfdev::ReplicaParams*>(ctx->args.rep), reps.data(),
                       reps.size() * sizeof(pfdev::ReplicaParams), cudaMemcpyHostToDevice));
    ctx->reps.swap(reps);
    ctx->rep_aps.swap(aps);
    set_skip_empty(ctx);
    set_cluster(ctx);
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);  // they captured the old StepArgs
    ctx->graphs.clear();
    ctx->graph_launches.clear();
    return PF_OK;
}

int32_t pf_replica_agents(const pf_ctx* ctx, int32_t rep) {
    if (!ctx || rep < 0 || rep >= ctx->cfg.replicas) return -1;
    return ctx->rep_aps[size_t(rep)];
}

// Global row of buffer row b.
static inline int64_t grow_of(const pf_ctx* ctx, int b) { return int64_t(ctx->row_begin) - pfk::kGhost + b; }

// Fused kernel: occupancy planes of both parities from the replica's words.
static void build_occ(pf_ctx* ctx, int rep) {
    pfk::Planes& P = ctx->args.p;
    if (!ctx->bits()) return;
    const size_t ooff = size_t(rep) * P.occ_plane;
    ctx->launches += pfk::launch_build_occ(P.cell[0] + size_t(rep) * ctx->plane(), ctx->cfg.width, ctx->rows_buf,
                                           P.wsp, P.occ[0] + ooff, P.occ[1] + ooff, ctx->stream);
}

// Fused kernel: zero the stale words of vacated cells (empty in the current
// planes) so the word plane is the exact cell-word state; *bad counts agent
// cells whose word disagrees with the planes. Owned rows only: on a linked
// row shard the neighbour's step kernel may still be storing words and plane
// bits into this shard's ghost rows (its stream is not ordered with ours), and
// every reader (export, audit) reads owned rows only.
static void sanitize_words(pf_ctx* ctx, int rep, unsigned long long* bad) {
    pfk::Planes& P = ctx->args.p;
    if (!ctx->bits()) return;
    const size_t W = size_t(ctx->cfg.width);
    ctx->launches += pfk::launch_sanitize_words(
        P.cell[0] + size_t(rep) * ctx->plane() + size_t(pfk::kGhost) * W,
        P.occ[ctx->parity] + size_t(rep) * P.occ_plane + size_t(pfk::kGhost) * P.wsp, ctx->cfg.width,
        ctx->rows_owned, P.wsp, bad, ctx->stream);
}

// Copy between aliased planes is a no-op.
static cudaError_t copy_d2d(void* dst, const void* src, size_t n, cudaStream_t s) {
    return dst == src ? cudaSuccess : cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s);
}

// Upload one replica's buffer-row planes (cells + tour) and set the step.
static int ensure_scratch(pf_ctx* ctx, size_t need);

// After replica rep's words are in P.cell[0] (pf_init_environment): the
// second word buffer, the occupancy planes, zero tours and the initial
// pheromone tau0 in both buffers (src/state.cpp:40-47).
static int finish_replica_init(pf_ctx* ctx, int rep) {
    const size_t off = size_t(rep) * ctx->plane();
    pfk::Planes& P = ctx->args.p;
    // The second ping-pong buffer is filled device-side (its ghost rows must
    // hold the same walls / halo).
    PF_CUDA(copy_d2d(P.cell[1] + off, P.cell[0] + off, ctx->plane() * 4, ctx->stream));
    build_occ(ctx, rep);
    if (ctx->aco()) {
        PF_CUDA(cudaMemsetAsync(P.tour + off, 0, ctx->plane() * 8, ctx->stream));
        ctx->launches += pfk::launch_fill_tau(ctx->tau_ptr(0, off), ctx->plane(), ctx->cfg.tau0, ctx->f32(), ctx->stream);
        ctx->launches += pfk::launch_fill_tau(ctx->tau_ptr(1, off), ctx->plane(), ctx->cfg.tau0, ctx->f32(), ctx->stream);
    }
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    return PF_OK;
}

static void set_step(pf_ctx* ctx, uint32_t step) {
    ctx->step = step;
    ctx->phase = 0;
    cudaMemcpyAsync(ctx->d_step, &ctx->step, 4, cudaMemcpyHostToDevice, ctx->stream);
    // Multi-step launches wait for tile_done >= their steps: no flag may be
    // ahead of the (possibly earlier) step the state is set to.
    if (ctx->args.tile_done) cudaMemsetAsync(ctx->args.tile_done, 0, ctx->tile_done_bytes, ctx->stream);
    if (ctx->linked) {  // linked neighbours are (re)loaded to the same step
        const uint32_t sync[2] = {step, step};
        cudaMemcpyAsync(ctx->d_sync, sync, 8, cudaMemcpyHostToDevice, ctx->stream);
    }
    cudaStreamSynchronize(ctx->stream);
}

int pf_init_environment(pf_ctx* ctx) {
    NvtxRange nvtx_range("pf_init_environment");
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    const pf_config& c = ctx->cfg;
    const uint32_t W = uint32_t(c.width);
    // new_environment (src/state.cpp:17-75): the placement (keyed
    // Fisher-Yates) is host work, cached per scenario and normally already
    // computed in the background since pf_create; replicas are independent,
    // so several are placed at once. Only the placed agents' cell lists go to
    // the device, where a kernel writes their words into a zeroed plane.
    const int R = c.replicas;
    const int nthreads = std::max(1, std::min<int>(R, int(std::thread::hardware_concurrency())));
    std::vector<std::shared_ptr<const pfhost::Placement>> pls(size_t(std::min(R, nthreads)));
    pfk::Planes& P = ctx->args.p;
    const int64_t g_lo = grow_of(ctx, 0);
    for (int r0 = 0; r0 < R; r0 += nthreads) {
        const int nb = std::min(nthreads, R - r0);
        std::atomic<bool> failed{false};
        std::vector<std::thread> ts;
        for (int t = 0; t < nb; ++t) {
            ts.emplace_back([&, t] {
                try {
                    pls[size_t(t)] = pfhost::placement(c.width, c.height, ctx->rep_aps[size_t(r0 + t)],
                                                       ctx->reps[size_t(r0 + t)].seed);
                } catch (...) {
                    failed = true;
                }
            });
        }
        for (auto& t : ts) t.join();
        if (failed) return fail(PF_ERR_CUDA, "new_environment: host allocation failed");
        for (int t = 0; t < nb; ++t) {
            const int rep = r0 + t;
            const size_t off = size_t(rep) * ctx->plane();
            const uint32_t n = uint32_t(ctx->rep_aps[size_t(rep)]);
            PF_CUDA(cudaMemsetAsync(P.cell[0] + off, 0, ctx->plane() * 4, ctx->stream));
            for (int b = 0; b < ctx->rows_buf; ++b) {  // rows outside the grid are walls
                const int64_t g = grow_of(ctx, b);
                if (g < 0 || g >= c.height)
                    PF_CUDA(cudaMemsetAsync(P.cell[0] + off + size_t(b) * W, 0xFF, size_t(W) * 4, ctx->stream));
            }
            if (n > 0) {
                if (int rc = ensure_scratch(ctx, size_t(n) * 8)) return rc;
                uint32_t* d_cells = static_cast<uint32_t*>(ctx->io_scratch);
                PF_CUDA(ctx->stage[0].h2d(d_cells, pls[size_t(t)]->cells[0].data(), size_t(n) * 4, ctx->stream));
                PF_CUDA(ctx->stage[0].h2d(d_cells + n, pls[size_t(t)]->cells[1].data(), size_t(n) * 4, ctx->stream));
                ctx->launches += pfk::launch_scatter_placement(P.cell[0] + off, d_cells, n, 1u, 1u, W, g_lo,
                                                               ctx->rows_buf, ctx->stream);
                ctx->launches += pfk::launch_scatter_placement(P.cell[0] + off, d_cells + n, n, n + 1u, 2u, W, g_lo,
                                                               ctx->rows_buf, ctx->stream);
            }
            if (int rc = finish_replica_init(ctx, rep)) return rc;
        }
    }
    ctx->parity = 0;
    set_step(ctx, 0);
    return PF_OK;
}

// Device scratch for state transfers, grown on demand and kept.
static int ensure_scratch(pf_ctx* ctx, size_t need) {
    if (ctx->io_scratch_bytes >= need) return PF_OK;
    if (ctx->io_scratch) cudaFree(ctx->io_scratch);
    ctx->io_scratch = nullptr;
    ctx->io_scratch_bytes = 0;
    PF_CUDA(cudaMalloc(&ctx->io_scratch, need));
    ctx->io_scratch_bytes = need;
    return PF_OK;
}

static size_t up256(size_t b) { return (b + 255) & ~size_t(255); }

int pf_load_state(pf_ctx* ctx, int32_t rep, const uint8_t* occ, const uint32_t* index, const pf_agent* agents,
                  uint32_t n_agents, const double* tau_top, const double* tau_bot, uint32_t step) {
    NvtxRange nvtx_range("pf_load_state");
    if (!ctx || !occ || !index) return fail(PF_ERR_ARG, "null argument");
    if (rep < 0 || rep >= ctx->cfg.replicas) return fail(PF_ERR_ARG, "replica out of range");
    const pf_config& c = ctx->cfg;
    if (n_agents != ctx->reps[size_t(rep)].n_agents) return fail(PF_ERR_STATE, "state corrupt: agent count disagrees with config");
    if (n_agents && !agents) return fail(PF_ERR_ARG, "null agents");
    if (ctx->aco() && (!tau_top || !tau_bot)) return fail(PF_ERR_ARG, "ACO state needs both pheromone fields");
    PF_CUDA(cudaSetDevice(c.device));
    PF_CUDA(cudaStreamSynchronize(ctx->stream));  // no step may still be using the planes
    IoTrace io_trace;
    const size_t W = size_t(c.width);
    const size_t off = size_t(rep) * ctx->plane();
    pfk::Planes& P = ctx->args.p;
    // The planes go up as they are (the reference's layout); the device checks
    // them and builds the cell words and the cell-resident tour. Rows of the
    // buffer window that lie inside the grid: [g_lo, g_hi).
    const int64_t g_lo = std::max<int64_t>(0, grow_of(ctx, 0));
    const int64_t g_hi = std::min<int64_t>(c.height, grow_of(ctx, ctx->rows_buf));
    const size_t b_lo = size_t(g_lo - grow_of(ctx, 0));
    const size_t win = size_t(g_hi - g_lo) * W;
    const size_t plane = ctx->plane();
    const size_t need = up256(win) + up256(win * 4) + up256(size_t(n_agents) * 40) + up256(plane * 4) +
                        (ctx->aco() ? up256(plane * 8) : 0) + (ctx->f32() ? up256(win * 16) : 0) + 16;
    if (int rc = ensure_scratch(ctx, need)) return rc;
    if (!ctx->io_event) PF_CUDA(cudaEventCreateWithFlags(&ctx->io_event, cudaEventDisableTiming));
    char* sp = static_cast<char*>(ctx->io_scratch);
    auto take = [&](size_t bytes) {
        char* p = sp;
        sp += up256(bytes);
        return p;
    };
    auto* d_occ = reinterpret_cast<uint8_t*>(take(win));
    auto* d_index = reinterpret_cast<uint32_t*>(take(win * 4));
    char* d_agents = take(size_t(n_agents) * 40);
    auto* d_words = reinterpret_cast<uint32_t*>(take(plane * 4));
    double* d_tour = ctx->aco() ? reinterpret_cast<double*>(take(plane * 8)) : nullptr;
    // Pheromone fields go up on a helper thread into the non-current ping-pong
    // buffer (scratch until the state is known to be valid).
    // (fp32 storage: the f64 fields go to the transfer scratch instead.)
    const int cur = ctx->parity;
    double* d_top = !ctx->aco() ? nullptr
                    : ctx->f32() ? reinterpret_cast<double*>(take(win * 16))
                                 : reinterpret_cast<double*>(P.tau[cur ^ 1] + off);
    double* d_bot = d_top ? d_top + (ctx->f32() ? win : plane) : nullptr;
    auto* d_status = reinterpret_cast<unsigned long long*>(sp);
    cudaError_t side_err = cudaSuccess;
    std::thread side;
    if (ctx->aco()) {
        side = std::thread([&] {
            cudaSetDevice(c.device);
            Stager& st = ctx->stage[1];
            cudaError_t e = st.h2d(d_top, tau_top + size_t(g_lo) * W, win * 8, ctx->stream2);
            if (e == cudaSuccess) e = st.h2d(d_bot, tau_bot + size_t(g_lo) * W, win * 8, ctx->stream2);
            if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream2);
            side_err = e;
        });
    }
    auto join_side = [&] {
        if (side.joinable()) side.join();
    };
    Stager& st = ctx->stage[0];
    cudaError_t e = st.h2d(d_occ, occ + size_t(g_lo) * W, win, ctx->stream);
    if (e == cudaSuccess) e = st.h2d(d_index, index + size_t(g_lo) * W, win * 4, ctx->stream);
    if (e == cudaSuccess && n_agents) e = st.h2d(d_agents, agents, size_t(n_agents) * 40, ctx->stream);
    io_trace("load: occupancy/index/agents up");
    // check_consistency-style audit (src/state.cpp:77-110) + conversion, on the device.
    unsigned long long status = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_status, &status, 8, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        ctx->launches += pfk::launch_import_state(d_occ, d_index, d_agents, n_agents, uint32_t(W), c.height,
                                                  grow_of(ctx, 0), g_lo, plane, d_words, d_tour, d_status,
                                                  ctx->stream);
        e = cudaMemcpyAsync(&status, d_status, 8, cudaMemcpyDeviceToHost, ctx->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    io_trace("load: device audit + conversion");
    if (e == cudaSuccess && status != ~0ull) {
        join_side();
        static const char* kWhy[] = {"", "state corrupt: index/occupancy mismatch",
                                     "state corrupt: index out of agent range", "state corrupt: agent record id mismatch",
                                     "state corrupt: agent position disagrees with index grid",
                                     "state corrupt: agent group disagrees with occupancy"};
        return fail(PF_ERR_STATE, kWhy[status & 7]);
    }
    // Valid: both ping-pong buffers receive the state (the parity is kept).
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(P.cell[cur] + off, d_words, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) e = copy_d2d(P.cell[cur ^ 1] + off, P.cell[cur] + off, plane * 4, ctx->stream);
    if (e == cudaSuccess) build_occ(ctx, rep);
    if (e == cudaSuccess && ctx->aco())
        e = cudaMemcpyAsync(P.tour + off, d_tour, plane * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    join_side();
    io_trace("load: side join (pheromone)");
    if (e == cudaSuccess) e = side_err;
    if (e == cudaSuccess && ctx->aco()) {
        // Interleave the two fields into {top, bottom} pairs (ghost rows
        // outside the grid hold zeros), then mirror into the scratch buffer.
        e = cudaMemsetAsync(ctx->tau_ptr(cur, off), 0, plane * ctx->tau_elem(), ctx->stream);
        ctx->launches += pfk::launch_interleave_tau(ctx->tau_ptr(cur, off + b_lo * W), d_top, d_bot, win, ctx->f32(),
                                                    ctx->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->tau_ptr(cur ^ 1, off), ctx->tau_ptr(cur, off), plane * ctx->tau_elem(),
                                cudaMemcpyDeviceToDevice, ctx->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail(PF_ERR_CUDA, std::string("state upload: ") + cudaGetErrorString(e));
    io_trace("load: device transforms");
    set_step(ctx, step);
    return PF_OK;
}

// Store of a whole (unsharded) grid: the device writes the reference planes
// (export_state_kernel, tau de-interleave), the host only copies them down,
// the pheromone fields on a helper thread.
static int store_whole(pf_ctx* ctx, int rep, uint8_t* occ, uint32_t* index, pf_agent* agents, uint32_t n_agents,
                       double* tau_top, double* tau_bot) {
    const pf_config& c = ctx->cfg;
    const size_t W = size_t(c.width);
    const size_t own = size_t(ctx->rows_owned) * W;
    const size_t off = size_t(rep) * ctx->plane() + size_t(pfk::kGhost) * W;
    const pfk::Planes& P = ctx->args.p;
    IoTrace io_trace;
    auto up = up256;
    const size_t need = up(own) + up(own * 4) + up(size_t(n_agents) * 40) + 24;
    if (int rc = ensure_scratch(ctx, need)) return rc;
    if (!ctx->io_event) PF_CUDA(cudaEventCreateWithFlags(&ctx->io_event, cudaEventDisableTiming));
    char* s = static_cast<char*>(ctx->io_scratch);
    auto* d_occ = reinterpret_cast<uint8_t*>(s);
    auto* d_index = reinterpret_cast<uint32_t*>(s + up(own));
    char* d_agents = s + up(own) + up(own * 4);
    auto* d_status = reinterpret_cast<unsigned long long*>(d_agents + up(size_t(n_agents) * 40));
    PF_CUDA(cudaMemsetAsync(d_status, 0, 24, ctx->stream));
    if (agents) PF_CUDA(cudaMemsetAsync(d_agents, 0, size_t(n_agents) * 40, ctx->stream));
    sanitize_words(ctx, rep, d_status + 2);
    const uint8_t* intents = ctx->phase >= 2 ? P.intent + off : nullptr;  // futures between intention and reset
    ctx->launches += pfk::launch_export_state(P.cell[ctx->parity] + off, ctx->aco() ? P.tour + off : nullptr, intents, own,
                                              uint32_t(W), uint32_t(ctx->row_begin), occ ? d_occ : nullptr,
                                              index ? d_index : nullptr, agents ? d_agents : nullptr, n_agents,
                                              d_status, ctx->stream);
    double* top = nullptr;
    if (ctx->aco() && (tau_top || tau_bot)) {
        // f64 scratch in the other ping-pong buffer (16 B per cell are allocated in both storage modes)
        top = reinterpret_cast<double*>(P.tau[ctx->parity ^ 1] + off);
        ctx->launches += pfk::launch_deinterleave_tau(top, top + own, ctx->tau_ptr(ctx->parity, off), own, ctx->f32(),
                                                      ctx->stream);
    }
    PF_CUDA(cudaEventRecord(ctx->io_event, ctx->stream));
    PF_CUDA(cudaStreamWaitEvent(ctx->stream2, ctx->io_event, 0));
    cudaError_t side_err = cudaSuccess;
    std::thread side;
    if (top) {
        side = std::thread([&] {
            cudaSetDevice(c.device);
            cudaError_t e = cudaSuccess;
            if (tau_top) e = ctx->stage[1].d2h(tau_top, top, own * 8, ctx->stream2);
            if (e == cudaSuccess && tau_bot) e = ctx->stage[1].d2h(tau_bot, top + own, own * 8, ctx->stream2);
            side_err = e;
        });
    }
    unsigned long long status[3] = {0, 0, 0};
    cudaError_t e = ctx->stage[0].d2h(status, d_status, 24, ctx->stream);
    if (e == cudaSuccess && occ) e = ctx->stage[0].d2h(occ, d_occ, own, ctx->stream);
    if (e == cudaSuccess && index) e = ctx->stage[0].d2h(index, d_index, own * 4, ctx->stream);
    if (e == cudaSuccess && agents) e = ctx->stage[0].d2h(agents, d_agents, size_t(n_agents) * 40, ctx->stream);
    io_trace("store: occ/index/agents down");
    if (side.joinable()) side.join();
    io_trace("store: side join (pheromone)");
    if (e == cudaSuccess) e = side_err;
    if (e != cudaSuccess) return fail(PF_ERR_CUDA, std::string("state download: ") + cudaGetErrorString(e));
    if (status[1]) return fail(PF_ERR_STATE, "state corrupt: device cell holds an out-of-range id");
    if (status[2]) return fail(PF_ERR_STATE, "state corrupt: cell words disagree with the occupancy planes");
    if (status[0] != n_agents) return fail(PF_ERR_STATE, "state corrupt: agents on the grid disagree with the agent count");
    return PF_OK;
}

int pf_store_state(pf_ctx* ctx, int32_t rep, uint8_t* occ, uint32_t* index, pf_agent* agents, uint32_t n_agents,
                   double* tau_top, double* tau_bot, uint32_t* step) {
    NvtxRange nvtx_range("pf_store_state");
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (rep < 0 || rep >= ctx->cfg.replicas) return fail(PF_ERR_ARG, "replica out of range");
    const pf_config& c = ctx->cfg;
    PF_CUDA(cudaSetDevice(c.device));
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->rows_owned == c.height && n_agents == ctx->reps[size_t(rep)].n_agents) {
        if (int rc = store_whole(ctx, rep, occ, index, agents, n_agents, tau_top, tau_bot)) return rc;
        if (step) *step = ctx->step;
        return PF_OK;
    }
    if (ctx->phase >= 2) return fail(PF_ERR_ARG, "a row shard's state cannot be stored in the middle of a phase-level step");
    IoTrace io_trace;
    const size_t W = size_t(c.width);
    const size_t own = size_t(ctx->rows_owned) * W;
    const size_t off = size_t(rep) * ctx->plane() + size_t(pfk::kGhost) * W;
    const pfk::Planes& P = ctx->args.p;
    std::unique_ptr<uint32_t[]> words_buf(new uint32_t[own]);
    uint32_t* words = words_buf.get();
    sanitize_words(ctx, rep, nullptr);
    PF_CUDA(ctx->stage[0].d2h(words, P.cell[ctx->parity] + off, own * 4, ctx->stream));
    const size_t g0 = size_t(ctx->row_begin) * W;
    // ACO: pheromone is de-interleaved on the device into the owned rows of
    // the other ping-pong buffer (rewritten by the next step anyway) and tour
    // lengths are gathered per agent (id order); a helper thread copies both
    // down while this thread converts the cell words.
    std::vector<double> per_agent;
    double* d_pa = nullptr;
    cudaError_t side_err = cudaSuccess;
    std::thread side;
    if (ctx->aco()) {
        per_agent.assign(n_agents, 0.0);
        PF_CUDA(cudaMalloc(&d_pa, std::max<size_t>(8, size_t(n_agents) * 8)));
        double* top = reinterpret_cast<double*>(P.tau[ctx->parity ^ 1] + off);
        double* bot = top + own;
        ctx->launches += pfk::launch_deinterleave_tau(top, bot, ctx->tau_ptr(ctx->parity, off), own, ctx->f32(),
                                                      ctx->stream);
        ctx->launches += pfk::launch_gather_tour(d_pa, P.cell[ctx->parity] + off, P.tour + off, own, ctx->stream);
        side = std::thread([&, top, bot] {
            cudaSetDevice(c.device);
            cudaError_t e = cudaSuccess;
            Stager& st = ctx->stage[1];
            if (tau_top) e = st.d2h(tau_top + g0, top, own * 8, ctx->stream);
            if (e == cudaSuccess && tau_bot) e = st.d2h(tau_bot + g0, bot, own * 8, ctx->stream);
            if (e == cudaSuccess) e = st.d2h(per_agent.data(), d_pa, size_t(n_agents) * 8, ctx->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
            side_err = e;
        });
    }
    std::atomic<bool> bad{false};
    io_trace("store: words down");
    host_parallel(own, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            const uint32_t w = words[i];
            const size_t gi = g0 + i;
            const uint32_t id = w & pfdev::kIdMask;
            if (occ) occ[gi] = uint8_t(w ? (w >> 30) : 0);
            if (index) index[gi] = w ? id : 0;
            if (!w) continue;
            if (id == 0 || id > n_agents) {
                bad = true;
                continue;
            }
            if (agents) {  // ids are unique, so the writes are disjoint
                pf_agent& a = agents[id - 1];
                std::memset(&a, 0, sizeof a);
                a.index = id;
                a.group = uint8_t(w >> 30);
                a.row = a.future_row = int32_t(gi / W);
                a.col = a.future_col = int32_t(gi % W);
                a.crossed = (w & pfdev::kCrossedBit) ? 1 : 0;
            }
        }
    });
    if (side.joinable()) side.join();
    io_trace("store: conversion + side join");
    cudaFree(d_pa);
    if (side_err != cudaSuccess) return fail(PF_ERR_CUDA, std::string("state download: ") + cudaGetErrorString(side_err));
    if (agents && ctx->aco() && !bad) {
        // Only agents on this shard's cells were gathered.
        host_parallel(own, [&](size_t i0, size_t i1) {
            for (size_t i = i0; i < i1; ++i)
                if (const uint32_t w = words[i]) agents[(w & pfdev::kIdMask) - 1].tour_length = per_agent[(w & pfdev::kIdMask) - 1];
        });
    }
    if (bad) return fail(PF_ERR_STATE, "state corrupt: device cell holds an out-of-range id");
    io_trace("store: tour fill");
    if (step) *step = ctx->step;
    return PF_OK;
}

// Zero the report-ring slots of steps [first, first + n) on every replica.
static int zero_reports(pf_ctx* ctx, uint32_t first, uint32_t n) {
    const size_t pitch = size_t(kReportCap) * 16;
    uint32_t done = 0;
    while (done < n) {
        const uint32_t slot = (first + done) % kReportCap;
        const uint32_t m = std::min<uint32_t>(n - done, kReportCap - slot);
        PF_CUDA(cudaMemset2DAsync(reinterpret_cast<char*>(ctx->d_reports) + size_t(slot) * 16, pitch, 0,
                                  size_t(m) * 16, size_t(ctx->cfg.replicas), ctx->stream));
        PF_CUDA(cudaMemsetAsync(ctx->args.bcount + size_t(slot) * 2, 0, size_t(m) * 8, ctx->stream));  // boundary items
        done += m;
    }
    // Work-item counters, one per batch slot (step_bits_kernel claims its
    // first item before griddepcontrol.wait, so they are not per step).
    PF_CUDA(cudaMemsetAsync(ctx->args.work, 0, size_t(std::min<uint32_t>(n, kBatchCap)) * 4, ctx->stream));
    return PF_OK;
}

static int launch_one_step(pf_ctx* ctx, uint32_t i, int parity) {
    // Linked shards: the step kernel itself orders its boundary items against
    // the neighbours' (wait_boundary / signal_boundary in pf_bitstep.cuh).
    switch (ctx->cfg.kernel) {
        case PF_KERNEL_FUSED:
        case PF_KERNEL_FUSED_F32: ctx->launches += pfk::launch_step_bits(ctx->args, int(i), parity, ctx->stream); break;
        case PF_KERNEL_TILE: ctx->launches += pfk::launch_step_fused(ctx->args, int(i), parity, ctx->stream); break;
        default: ctx->launches += pfk::launch_step_pipeline(ctx->args, int(i), parity, ctx->stream); break;
    }
    return PF_OK;
}

// Steps are stream-ordered; a handshake timeout (a neighbour that never
// completed its step) is reported at the next synchronisation.
static int check_halo(pf_ctx* ctx) {
    if (!ctx->linked && !ctx->multistep) return PF_OK;
    uint32_t err = 0;
    PF_CUDA(cudaMemcpy(&err, ctx->d_err, 4, cudaMemcpyDeviceToHost));
    if (err & 1u) return fail(PF_ERR_COMM, "fused halo exchange: a neighbour shard did not complete its step (timeout)");
    if (err & 2u) return fail(PF_ERR_CUDA, "multi-step launch: a tile dependency wait timed out (internal error)");
    if (err & 4u) return fail(PF_ERR_CUDA, "cluster-resident LEM kernel: a work list overflowed (internal error)");
    return PF_OK;
}

// Enqueue n <= kBatchCap steps (batch slots 0..n-1) with the given start
// parity: one multi-step launch (PF_KERNEL_FUSED, unlinked contexts: steps
// overlap at tile granularity, pf_bitstep.cuh) or one launch per step.
static int enqueue_direct(pf_ctx* ctx, uint32_t n, int parity) {
    if (ctx->bits() && ctx->multistep && !ctx->linked && n > 1) {
        pfk::StepArgs b = ctx->args;
        b.nsteps = int(n);
        ctx->launches += pfk::launch_step_bits(b, 0, parity, ctx->stream);
    } else {
        for (uint32_t i = 0; i < n; ++i) launch_one_step(ctx, i, (parity + int(i)) & 1);
    }
    ctx->launches += pfk::launch_advance_step(ctx->d_step, n, ctx->stream);
    return PF_OK;
}

// The cached graph of n steps starting at the given parity (captured and
// instantiated on first use).
static int batch_graph(pf_ctx* ctx, uint32_t n, int parity, cudaGraphExec_t* out) {
    const auto key = std::make_pair(n, parity);
    auto it = ctx->graphs.find(key);
    if (it == ctx->graphs.end()) {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        const uint64_t before = ctx->launches;
        PF_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        enqueue_direct(ctx, n, parity);
        PF_CUDA(cudaStreamEndCapture(ctx->stream, &g));
        ctx->graph_launches[key] = ctx->launches - before;
        ctx->launches = before;  // counted when replayed
        PF_CUDA(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        it = ctx->graphs.emplace(key, ge).first;
    }
    *out = it->second;
    return PF_OK;
}

int pf_prepare_steps(pf_ctx* ctx, uint32_t n) {
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    int parity = ctx->parity;
    while (n > 0) {
        const uint32_t m = std::min<uint32_t>(n, kBatchCap);
        cudaGraphExec_t ge = nullptr;
        if (int rc = batch_graph(ctx, m, parity, &ge)) return rc;
        parity ^= int(m & 1u);
        n -= m;
    }
    return PF_OK;
}

static int enqueue_batch(pf_ctx* ctx, uint32_t n) {
    if (int rc = zero_reports(ctx, ctx->step, n)) return rc;
    cudaGraphExec_t ge = nullptr;
    if (int rc = batch_graph(ctx, n, ctx->parity, &ge)) return rc;
    PF_CUDA(cudaGraphLaunch(ge, ctx->stream));
    ctx->launches += ctx->graph_launches[std::make_pair(n, ctx->parity)];
    ctx->parity ^= int(n & 1u);
    ctx->step += n;
    PF_CUDA(cudaGetLastError());
    return PF_OK;
}

int pf_step_async(pf_ctx* ctx, uint32_t n) {
    NvtxRange nvtx_range("pf_step_async");
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (ctx->phase) return fail(PF_ERR_ARG, "a phase-level step is in progress: finish it with PF_PHASE_RESET");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    while (n > 0) {
        const uint32_t m = std::min<uint32_t>(n, kBatchCap);
        if (int rc = enqueue_batch(ctx, m)) return rc;
        n -= m;
    }
    return PF_OK;
}

// Reports of the last n steps ([step - n, step)) of every replica: out is
// [replicas][n].
int pf_read_reports(pf_ctx* ctx, pf_step_report* out, uint32_t n) {
    if (!ctx || (!out && n)) return fail(PF_ERR_ARG, "null argument");
    if (n > uint32_t(kReportCap)) return fail(PF_ERR_ARG, "at most 1024 step reports are kept on the device");
    if (n > ctx->step) return fail(PF_ERR_ARG, "fewer steps than requested reports");
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    const int R = ctx->cfg.replicas;
    const size_t pitch = size_t(kReportCap) * 16;
    const uint32_t first = ctx->step - n;
    uint32_t done = 0;
    while (done < n) {
        const uint32_t slot = (first + done) % kReportCap;
        const uint32_t m = std::min<uint32_t>(n - done, kReportCap - slot);
        PF_CUDA(cudaMemcpy2D(out + done, size_t(n) * 16, reinterpret_cast<const char*>(ctx->d_reports) + size_t(slot) * 16,
                             pitch, size_t(m) * 16, size_t(R), cudaMemcpyDeviceToHost));
        done += m;
    }
    return PF_OK;
}

int pf_synchronize(pf_ctx* ctx) {
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    return check_halo(ctx);
}

int pf_step(pf_ctx* ctx, uint32_t n, pf_step_report* out) {
    NvtxRange nvtx_range("pf_step");
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (ctx->phase) return fail(PF_ERR_ARG, "a phase-level step is in progress: finish it with PF_PHASE_RESET");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    const int R = ctx->cfg.replicas;
    std::vector<pf_step_report> chunk;
    uint32_t done = 0;
    while (done < n) {
        const uint32_t m = std::min<uint32_t>(n - done, kBatchCap);
        if (int rc = enqueue_batch(ctx, m)) return rc;
        if (out) {
            chunk.resize(size_t(R) * m);
            if (int rc = pf_read_reports(ctx, chunk.data(), m)) return rc;
            for (int r = 0; r < R; ++r)
                std::memcpy(out + size_t(r) * n + done, chunk.data() + size_t(r) * m, size_t(m) * 16);
        }
        done += m;
    }
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    return check_halo(ctx);
}

int pf_time_steps(pf_ctx* ctx, uint32_t n, float* total_ms, float* kernel_ms) {
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (ctx->phase) return fail(PF_ERR_ARG, "a phase-level step is in progress: finish it with PF_PHASE_RESET");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    cudaEvent_t e0, e1;
    PF_CUDA(cudaEventCreate(&e0));
    PF_CUDA(cudaEventCreate(&e1));
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    PF_CUDA(cudaEventRecord(e0, ctx->stream));
    if (int rc = pf_step_async(ctx, n)) return rc;
    PF_CUDA(cudaEventRecord(e1, ctx->stream));
    PF_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (total_ms) *total_ms = ms;
    if (kernel_ms) {
        // Per-launch events around each step's kernel(s), no graph.
        std::vector<cudaEvent_t> ev(2 * size_t(n));
        for (auto& e : ev) PF_CUDA(cudaEventCreate(&e));
        uint32_t done = 0;
        while (done < n) {
            const uint32_t m = std::min<uint32_t>(n - done, kBatchCap);
            if (int rc = zero_reports(ctx, ctx->step, m)) return rc;
            for (uint32_t i = 0; i < m; ++i) {
                PF_CUDA(cudaEventRecord(ev[2 * (done + i)], ctx->stream));
                launch_one_step(ctx, i, (ctx->parity + int(i)) & 1);
                PF_CUDA(cudaEventRecord(ev[2 * (done + i) + 1], ctx->stream));
            }
            ctx->launches += pfk::launch_advance_step(ctx->d_step, m, ctx->stream);
            ctx->parity ^= int(m & 1u);
            ctx->step += m;
            done += m;
        }
        PF_CUDA(cudaStreamSynchronize(ctx->stream));
        double sum = 0.0;
        for (uint32_t i = 0; i < n; ++i) {
            float t = 0.f;
            PF_CUDA(cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]));
            sum += t;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        *kernel_ms = n ? float(sum / n) : 0.f;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return PF_OK;
}

uint32_t pf_current_step(const pf_ctx* ctx) { return ctx ? ctx->step : 0; }
void* pf_stream(pf_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
uint64_t pf_launch_count(const pf_ctx* ctx) { return ctx ? ctx->launches : 0; }

int pf_halo(pf_ctx* ctx, int32_t rep, int32_t side, int32_t recv, pf_halo_rows* out) {
    if (!ctx || !out) return fail(PF_ERR_ARG, "null argument");
    if (rep < 0 || rep >= ctx->cfg.replicas || (side != 0 && side != 1) || (recv != 0 && recv != 1))
        return fail(PF_ERR_ARG, "bad halo selector");
    const size_t W = size_t(ctx->cfg.width);
    const int G = pfk::kGhost;
    int first, tour_row;
    if (side == 0) {
        first = recv ? 0 : G;
        tour_row = recv ? G - 1 : G;
    } else {
        first = recv ? G + ctx->rows_owned : ctx->rows_owned;  // owned rows [rows_owned, rows_owned+G) in buffer = last G owned
        tour_row = recv ? G + ctx->rows_owned : G + ctx->rows_owned - 1;
    }
    const size_t off = size_t(rep) * ctx->plane();
    const pfk::Planes& P = ctx->args.p;
    out->cells = P.cell[ctx->parity] + off + size_t(first) * W;
    out->cell_bytes = size_t(G) * W * 4;
    if (ctx->bits()) {
        out->occ = P.occ[ctx->parity] + size_t(rep) * P.occ_plane + size_t(first) * P.wsp;
        out->occ_bytes = size_t(G) * P.wsp * 8;
    } else {
        out->occ = nullptr;
        out->occ_bytes = 0;
    }
    if (ctx->aco()) {
        out->tau = ctx->tau_ptr(ctx->parity, off + size_t(first) * W);
        out->tau_bytes = size_t(G) * W * ctx->tau_elem();
        out->tour = P.tour + off + size_t(tour_row) * W;
        out->tour_bytes = W * 8;
    } else {
        out->tau = out->tour = nullptr;
        out->tau_bytes = out->tour_bytes = 0;
    }
    return PF_OK;
}

int pf_exchange_pair(pf_ctx* upper, pf_ctx* lower) {
    if (!upper || !lower) return fail(PF_ERR_ARG, "null ctx");
    if (upper->cfg.replicas != lower->cfg.replicas || upper->cfg.width != lower->cfg.width ||
        upper->row_begin + upper->rows_owned != lower->row_begin)
        return fail(PF_ERR_COMM, "shards are not vertically adjacent");
    PF_CUDA(cudaSetDevice(upper->cfg.device));
    PF_CUDA(cudaStreamSynchronize(upper->stream));
    PF_CUDA(cudaSetDevice(lower->cfg.device));
    PF_CUDA(cudaStreamSynchronize(lower->stream));
    for (int r = 0; r < upper->cfg.replicas; ++r) {
        pf_halo_rows us, ur, ls, lr;
        pf_halo(upper, r, 1, 0, &us);
        pf_halo(upper, r, 1, 1, &ur);
        pf_halo(lower, r, 0, 0, &ls);
        pf_halo(lower, r, 0, 1, &lr);
        PF_CUDA(cudaMemcpyAsync(lr.cells, us.cells, us.cell_bytes, cudaMemcpyDefault, lower->stream));
        PF_CUDA(cudaMemcpyAsync(ur.cells, ls.cells, ls.cell_bytes, cudaMemcpyDefault, lower->stream));
        if (us.occ && ls.occ && us.occ_bytes == lr.occ_bytes) {
            PF_CUDA(cudaMemcpyAsync(lr.occ, us.occ, us.occ_bytes, cudaMemcpyDefault, lower->stream));
            PF_CUDA(cudaMemcpyAsync(ur.occ, ls.occ, ls.occ_bytes, cudaMemcpyDefault, lower->stream));
        } else if (us.occ || ls.occ) {
            return fail(PF_ERR_COMM, "shards use different kernels");
        }
        if (us.tau) {
            PF_CUDA(cudaMemcpyAsync(lr.tau, us.tau, us.tau_bytes, cudaMemcpyDefault, lower->stream));
            PF_CUDA(cudaMemcpyAsync(ur.tau, ls.tau, ls.tau_bytes, cudaMemcpyDefault, lower->stream));
            PF_CUDA(cudaMemcpyAsync(lr.tour, us.tour, us.tour_bytes, cudaMemcpyDefault, lower->stream));
            PF_CUDA(cudaMemcpyAsync(ur.tour, ls.tour, ls.tour_bytes, cudaMemcpyDefault, lower->stream));
        }
    }
    PF_CUDA(cudaStreamSynchronize(lower->stream));
    return PF_OK;
}

int pf_phase(pf_ctx* ctx, int32_t phase, pf_step_report* out) {
    NvtxRange nvtx_range("pf_phase");
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (ctx->cfg.kernel != PF_KERNEL_PIPELINE)
        return fail(PF_ERR_CONFIG, "phase-level stepping needs PF_KERNEL_PIPELINE (the fused kernels run all four phases "
                                   "in one launch)");
    if (phase < PF_PHASE_SCORE || phase > PF_PHASE_RESET) return fail(PF_ERR_ARG, "unknown phase");
    if (phase != ctx->phase)
        return fail(PF_ERR_ARG, "phases must run in order: score, intention, movement, reset");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    const int R = ctx->cfg.replicas;
    switch (phase) {
        case PF_PHASE_SCORE: {  // src/engine.cpp:64-74
            uint32_t n_max = 0;
            for (const auto& r : ctx->reps) n_max = std::max(n_max, r.n_agents);
            n_max = std::max(n_max, 1u);
            if (ctx->scores_n < n_max) {
                if (ctx->d_scores) cudaFree(ctx->d_scores);
                ctx->d_scores = nullptr;
                ctx->scores_n = 0;
                PF_CUDA(cudaMalloc(&ctx->d_scores, size_t(R) * n_max * 64));
                ctx->scores_n = n_max;
            }
            PF_CUDA(cudaMemsetAsync(ctx->d_scores, 0, size_t(R) * ctx->scores_n * 64, ctx->stream));
            ctx->launches += pfk::launch_score_phase(ctx->args, ctx->parity, ctx->d_scores, nullptr, ctx->scores_n,
                                                     ctx->stream);
            break;
        }
        case PF_PHASE_INTENTION:  // src/engine.cpp:76-90
            ctx->launches += pfk::launch_intention_phase(ctx->args, ctx->parity, ctx->stream);
            break;
        case PF_PHASE_MOVEMENT: {  // src/engine.cpp:92-180
            if (int rc = zero_reports(ctx, ctx->step, 1)) return rc;
            ctx->launches += pfk::launch_movement_phase(ctx->args, ctx->parity, ctx->stream);
            ctx->parity ^= 1;
            if (out) {
                const size_t pitch = size_t(kReportCap) * 16;
                PF_CUDA(cudaMemcpy2DAsync(out, 16, reinterpret_cast<const char*>(ctx->d_reports) +
                                                       size_t(ctx->step % kReportCap) * 16,
                                          pitch, 16, size_t(R), cudaMemcpyDeviceToHost, ctx->stream));
            }
            break;
        }
        default:  // PF_PHASE_RESET, src/engine.cpp:183-193: scores zeroed, futures = positions, ++step
            if (ctx->d_scores) PF_CUDA(cudaMemsetAsync(ctx->d_scores, 0, size_t(R) * ctx->scores_n * 64, ctx->stream));
            ctx->launches += pfk::launch_advance_step(ctx->d_step, 1, ctx->stream);
            ++ctx->step;
            break;
    }
    PF_CUDA(cudaGetLastError());
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->phase = phase == PF_PHASE_RESET ? 0 : phase + 1;
    return PF_OK;
}

int pf_store_scores(pf_ctx* ctx, int32_t rep, double* scores, uint32_t* owners, uint32_t n_agents) {
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (rep < 0 || rep >= ctx->cfg.replicas) return fail(PF_ERR_ARG, "replica out of range");
    if (n_agents != ctx->reps[size_t(rep)].n_agents) return fail(PF_ERR_ARG, "agent count disagrees with the replica");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    // owner is always the agent's id: set by new_environment (src/state.cpp:48)
    // and by every score_phase, never cleared (src/engine.cpp:183-193).
    if (owners)
        for (uint32_t i = 0; i < n_agents; ++i) owners[i] = i + 1;
    if (!scores || !n_agents) return PF_OK;
    if (!ctx->d_scores) {  // never scored: zeros, as new_environment leaves them
        std::memset(scores, 0, size_t(n_agents) * 64);
        return PF_OK;
    }
    PF_CUDA(cudaMemcpy(scores, ctx->d_scores + size_t(rep) * ctx->scores_n * 8, size_t(n_agents) * 64,
                       cudaMemcpyDeviceToHost));
    return PF_OK;
}

void* pf_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        g_err = "cudaHostAlloc failed";
        return nullptr;
    }
    return p;
}

int pf_host_free(void* p) {
    if (p) PF_CUDA(cudaFreeHost(p));
    return PF_OK;
}

int pf_peer_export(pf_ctx* ctx, pf_peer_desc* out) {
    if (!ctx || !out) return fail(PF_ERR_ARG, "null argument");
    if (!ctx->bits()) return fail(PF_ERR_CONFIG, "the fused halo exchange needs PF_KERNEL_FUSED");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    std::memset(out, 0, sizeof *out);
    const pfk::Planes& P = ctx->args.p;
    void* ptrs[7] = {P.cell[0], P.occ[0], P.occ[1], P.tau[0], P.tau[1], P.tour, ctx->d_sync};
    for (int i = 0; i < 7; ++i) {
        out->ptr[i] = reinterpret_cast<uint64_t>(ptrs[i]);
        if (!ptrs[i]) continue;
        cudaIpcMemHandle_t h;
        PF_CUDA(cudaIpcGetMemHandle(&h, ptrs[i]));
        static_assert(sizeof h == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(out->ipc[i], &h, 64);
    }
    out->device = ctx->cfg.device;
    out->width = ctx->cfg.width;
    out->replicas = ctx->cfg.replicas;
    out->model = ctx->cfg.model;
    out->kernel = ctx->cfg.kernel;
    out->row_begin = ctx->row_begin;
    out->rows_owned = ctx->rows_owned;
    out->parity = ctx->parity;
    out->step = ctx->step;
    out->plane = ctx->plane();
    out->occ_plane = P.occ_plane;
    return PF_OK;
}

int pf_peer_attach(pf_ctx* ctx, int32_t side, const pf_peer_desc* d, int32_t ipc) {
    if (!ctx || !d) return fail(PF_ERR_ARG, "null argument");
    if (side != 0 && side != 1) return fail(PF_ERR_ARG, "side must be 0 (above) or 1 (below)");
    if (!ctx->bits() || d->kernel != ctx->cfg.kernel)
        return fail(PF_ERR_CONFIG, "the fused halo exchange needs PF_KERNEL_FUSED (or _F32) on both sides");
    if (d->width != ctx->cfg.width || d->replicas != ctx->cfg.replicas || d->model != ctx->cfg.model)
        return fail(PF_ERR_COMM, "neighbour shard has a different grid width, replica count or model");
    const bool adjacent = side == 0 ? d->row_begin + d->rows_owned == ctx->row_begin
                                    : ctx->row_begin + ctx->rows_owned == d->row_begin;
    if (!adjacent) return fail(PF_ERR_COMM, "shards are not vertically adjacent");
    if (d->step != ctx->step || d->parity != ctx->parity)
        return fail(PF_ERR_COMM, "neighbour shard is at a different step");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    PF_CUDA(cudaStreamSynchronize(ctx->stream));
    void* p[7] = {};
    for (int i = 0; i < 7; ++i) {
        if (!d->ptr[i]) continue;
        if (ipc) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, d->ipc[i], 64);
            PF_CUDA(cudaIpcOpenMemHandle(&p[i], h, cudaIpcMemLazyEnablePeerAccess));
            ctx->ipc_opened.push_back(p[i]);
        } else {
            p[i] = reinterpret_cast<void*>(d->ptr[i]);
        }
    }
    if (!ipc && d->device != ctx->cfg.device) {
        int can = 0;
        PF_CUDA(cudaDeviceCanAccessPeer(&can, ctx->cfg.device, d->device));
        if (!can) return fail(PF_ERR_COMM, "no peer access between the shards' devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(d->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(PF_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        cudaGetLastError();
    }
    pfk::PeerRows& pr = ctx->args.peer[side];
    pr.cell = static_cast<uint32_t*>(p[0]);
    pr.occ[0] = static_cast<uint2*>(p[1]);
    pr.occ[1] = static_cast<uint2*>(p[2]);
    pr.tau[0] = static_cast<double2*>(p[3]);
    pr.tau[1] = static_cast<double2*>(p[4]);
    pr.tour = static_cast<double*>(p[5]);
    pr.plane = size_t(d->plane);
    pr.occ_plane = size_t(d->occ_plane);
    // Our owned row r (buffer row G + r) is the upper neighbour's lower ghost
    // row G + its rows_owned + r, and the lower neighbour's upper ghost row
    // r - (rows_owned - G).
    pr.row_delta = side == 0 ? d->rows_owned : -ctx->rows_owned;
    ctx->remote_flag[side] = static_cast<uint32_t*>(p[6]) + (1 - side);
    ctx->args.sync_remote[side] = ctx->remote_flag[side];
    if (d->device == ctx->cfg.device) ctx->args.peer_same_device = 1;
    const uint32_t now = ctx->step;  // the neighbour has completed `step` steps
    PF_CUDA(cudaMemcpy(ctx->d_sync + side, &now, 4, cudaMemcpyHostToDevice));
    ctx->linked |= 1 << side;
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);  // recaptured with the handshake
    ctx->graphs.clear();
    ctx->graph_launches.clear();
    return PF_OK;
}

int pf_audit(pf_ctx* ctx, int32_t rep, uint64_t* agent_cells) {
    NvtxRange nvtx_range("pf_audit");
    if (!ctx) return fail(PF_ERR_ARG, "null ctx");
    if (rep < 0 || rep >= ctx->cfg.replicas) return fail(PF_ERR_ARG, "replica out of range");
    PF_CUDA(cudaSetDevice(ctx->cfg.device));
    const uint32_t n_agents = ctx->reps[size_t(rep)].n_agents;
    const size_t words = (size_t(n_agents) + 31) / 32;
    char* d = nullptr;
    PF_CUDA(cudaMalloc(&d, words * 4 + 4 * 8));
    auto* counts = reinterpret_cast<unsigned long long*>(d);
    auto* seen = reinterpret_cast<uint32_t*>(d + 4 * 8);
    unsigned long long h[4] = {0ull, 0ull, ~0ull, 0ull};
    int rc = PF_OK;
    if (cudaMemcpyAsync(counts, h, sizeof h, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(seen, 0, words * 4, ctx->stream) != cudaSuccess) {
        rc = fail(PF_ERR_CUDA, "audit setup failed");
    } else {
        const size_t W = size_t(ctx->cfg.width);
        sanitize_words(ctx, rep, counts + 3);
        ctx->launches += pfk::launch_audit(ctx->args.p.cell[ctx->parity] + size_t(rep) * ctx->plane(),
                                           size_t(pfk::kGhost) * W, size_t(ctx->rows_owned) * W, n_agents, seen,
                                           counts, ctx->stream);
        if (cudaMemcpyAsync(h, counts, sizeof h, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = fail(PF_ERR_CUDA, "audit failed");
    }
    cudaFree(d);
    if (rc) return rc;
    if (agent_cells) *agent_cells = h[0];
    if (h[3]) return fail(PF_ERR_STATE, "state corrupt: " + std::to_string(h[3]) + " cell word(s) disagree with the occupancy planes");
    if (h[1]) {
        const size_t cell = size_t(h[2] - 1);
        const size_t W = size_t(ctx->cfg.width);
        return fail(PF_ERR_STATE, "state corrupt: " + std::to_string(h[1]) + " bad cell(s), first at (" +
                                      std::to_string(ctx->row_begin + cell / W) + "," + std::to_string(cell % W) + ")");
    }
    // A single (unsharded) context must hold every agent exactly once.
    if (ctx->rows_owned == ctx->cfg.height && h[0] != n_agents)
        return fail(PF_ERR_STATE, "state corrupt: agent count disagrees with occupied cells");
    return PF_OK;
}

int pf_selftest_select(int32_t device, int32_t kind, uint32_t n, double d0, double sel_mu, double sel_sigma,
                       const uint8_t* mask, const double* num, const uint64_t* seed, const uint32_t* step,
                       const uint64_t* entity, int32_t* out) {
    if (kind < 0 || kind > 2) return fail(PF_ERR_ARG, "kind must be 0 (lem), 1 (aco) or 2 (resolve)");
    if (!mask || !seed || !step || !entity || !out || (kind == 1 && !num)) return fail(PF_ERR_ARG, "null array");
    if (!(d0 > 1.0)) return fail(PF_ERR_CONFIG, "d0 must be > 1");
    if (n == 0) return PF_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PF_ERR_CUDA, "no CUDA device available");
    PF_CUDA(cudaSetDevice(device));
    pf_ctx tmp;  // only for fill_consts: the scores / factors exactly as a context computes them
    tmp.cfg.d0 = d0;
    tmp.cfg.sel_mu = sel_mu;
    tmp.cfg.sel_sigma = sel_sigma;
    tmp.cfg.alpha = 1.0;
    tmp.cfg.beta = 2.0;
    tmp.cfg.rho = 0.05;
    tmp.cfg.q = 1.0;
    tmp.cfg.model = kind == 1 ? PF_MODEL_ACO : PF_MODEL_LEM;
    fill_consts(&tmp);
    const size_t bytes = sizeof(pfdev::StepConsts) + size_t(n) * (1 + 8 + 4 + 8 + 4) + (num ? size_t(n) * 64 : 0) + 64;
    char* d = nullptr;
    PF_CUDA(cudaMalloc(&d, bytes));
    auto* d_kc = reinterpret_cast<pfdev::StepConsts*>(d);
    auto* d_seed = reinterpret_cast<uint64_t*>(d + ((sizeof(pfdev::StepConsts) + 15) & ~size_t(15)));
    uint64_t* d_ent = d_seed + n;
    double* d_num = reinterpret_cast<double*>(d_ent + n);
    uint32_t* d_step = reinterpret_cast<uint32_t*>(d_num + (num ? size_t(n) * 8 : 0));
    int32_t* d_out = reinterpret_cast<int32_t*>(d_step + n);
    uint8_t* d_mask = reinterpret_cast<uint8_t*>(d_out + n);
    auto run = [&]() -> int {
        PF_CUDA(cudaMemcpy(d_kc, &tmp.args.k, sizeof(pfdev::StepConsts), cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_seed, seed, n * 8, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_ent, entity, n * 8, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_step, step, n * 4, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_mask, mask, n, cudaMemcpyHostToDevice));
        if (num) PF_CUDA(cudaMemcpy(d_num, num, size_t(n) * 64, cudaMemcpyHostToDevice));
        pfk::launch_selftest_select(kind, n, d_kc, d_mask, num ? d_num : nullptr, d_seed, d_step, d_ent, d_out, 0);
        PF_CUDA(cudaGetLastError());
        PF_CUDA(cudaDeviceSynchronize());
        PF_CUDA(cudaMemcpy(out, d_out, n * 4, cudaMemcpyDeviceToHost));
        return PF_OK;
    };
    const int rc = run();
    cudaFree(d);
    return rc;
}

int pf_selftest_rng(int32_t device, uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                    const uint64_t* entity, const uint32_t* counter, double mu, double sigma, uint64_t* bits_out,
                    double* uniform_out, double* normal_out) {
    if (!seed || !step || !phase || !entity || !counter) return fail(PF_ERR_ARG, "null key array");
    if (n == 0) return PF_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PF_ERR_CUDA, "no CUDA device available");
    PF_CUDA(cudaSetDevice(device));
    const size_t in_bytes = size_t(n) * (8 + 4 + 4 + 8 + 4), out_bytes = size_t(n) * 24;
    char* d = nullptr;
    PF_CUDA(cudaMalloc(&d, in_bytes + out_bytes));
    uint64_t* d_seed = reinterpret_cast<uint64_t*>(d);
    uint64_t* d_ent = d_seed + n;
    uint64_t* d_bits = d_ent + n;
    double* d_uni = reinterpret_cast<double*>(d_bits + n);
    double* d_nrm = d_uni + n;
    uint32_t* d_step = reinterpret_cast<uint32_t*>(d_nrm + n);
    uint32_t* d_phase = d_step + n;
    uint32_t* d_ctr = d_phase + n;
    auto run = [&]() -> int {
        PF_CUDA(cudaMemcpy(d_seed, seed, n * 8, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_ent, entity, n * 8, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_step, step, n * 4, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_phase, phase, n * 4, cudaMemcpyHostToDevice));
        PF_CUDA(cudaMemcpy(d_ctr, counter, n * 4, cudaMemcpyHostToDevice));
        pfk::launch_selftest_rng(n, d_seed, d_step, d_phase, d_ent, d_ctr, mu, sigma, d_bits, d_uni, d_nrm, 0);
        PF_CUDA(cudaGetLastError());
        PF_CUDA(cudaDeviceSynchronize());
        if (bits_out) PF_CUDA(cudaMemcpy(bits_out, d_bits, n * 8, cudaMemcpyDeviceToHost));
        if (uniform_out) PF_CUDA(cudaMemcpy(uniform_out, d_uni, n * 8, cudaMemcpyDeviceToHost));
        if (normal_out) PF_CUDA(cudaMemcpy(normal_out, d_nrm, n * 8, cudaMemcpyDeviceToHost));
        return PF_OK;
    };
    const int rc = run();
    cudaFree(d);
    return rc;
}

}  // extern "C"
