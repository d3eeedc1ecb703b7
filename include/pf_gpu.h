/* pf_gpu.h — C-ABI of the B200-native per-step grid update (pedflow-b200).
 *
 * Drop-in boundary for the reference's hot path: the C++ class
 * pedflow::StepEngine (/root/reference/proj/include/pedflow/engine.hpp:48-66)
 * and its setup call new_environment (include/pedflow/state.hpp:37). The
 * reference has no FFI; this header is what a binding to that path needs:
 * plain pointers and sizes, no exceptions, no C++ or torch types. The C++
 * shim include/pedflow_gpu.hpp re-exposes it as pedflow::gpu::StepEngine.
 *
 * Status codes mirror the reference's error classes (inc/errors.hpp:9-11,
 * tools/pedflow.cpp:253-258): PF_ERR_CONFIG is ConfigError; PF_ERR_STATE is
 * the std::logic_error("state corrupt: ...") of check_consistency
 * (src/state.cpp:77-110). pf_last_error() gives the message (thread-local).
 */
#ifndef PF_GPU_H
#define PF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_ERR_CONFIG 2 /* ConfigError: invalid scenario parameters */
#define PF_ERR_CUDA 3   /* CUDA runtime failure (no device, OOM, launch error) */
#define PF_ERR_COMM 4   /* halo exchange failure */
#define PF_ERR_STATE 5  /* state corrupt: inconsistent planes passed to pf_load_state */
#define PF_ERR_ARG 6    /* bad argument (null pointer, replica out of range) */

#define PF_MODEL_LEM 0
#define PF_MODEL_ACO 1

#define PF_KERNEL_FUSED 0    /* one bit-sliced kernel per step on occupancy bit planes (default) */
#define PF_KERNEL_PIPELINE 1 /* propose / resolve / commit, three kernels per step */
#define PF_KERNEL_TILE 2     /* one kernel per step, scalar per-cell shared-memory tile */
#define PF_KERNEL_FUSED_F32 3 /* PF_KERNEL_FUSED with the ACO pheromone stored as fp32 (arithmetic still
                               * fp64, one rounding per store): half the pheromone traffic,
                               * tolerance-only parity; LEM runs as PF_KERNEL_FUSED */

/* Number of ghost rows kept above and below a row shard: one step's
 * dependency radius. */
#define PF_GHOST_ROWS 3

/* ScenarioConfig numerics (inc/config.hpp:20-58) + the GPU's additions.
 * replaces: pedflow::ScenarioConfig + EngineOptions::from_config
 * (src/engine.cpp:35-46). */
typedef struct pf_config {
    int32_t width, height, agents_per_side, model;
    uint64_t seed; /* replica i runs seed + i (tools/pedflow.cpp:135 repeat schedule) */
    double d0, sel_mu, sel_sigma, alpha, beta, rho, tau0, q;
    int32_t replicas;  /* >= 1 independent scenarios stepped by one launch */
    int32_t row_begin; /* owned global rows [row_begin, row_end) of a row shard; */
    int32_t row_end;   /* row_end == 0 means the whole grid */
    int32_t device;    /* CUDA device ordinal */
    int32_t kernel;    /* PF_KERNEL_FUSED, PF_KERNEL_PIPELINE, PF_KERNEL_TILE or PF_KERNEL_FUSED_F32 */
} pf_config;

/* Byte-identical to pedflow::AgentRecord (inc/grid.hpp:84-93), 40 bytes. */
typedef struct pf_agent {
    uint32_t index; /* 1-based id */
    uint8_t group;  /* 1 Top, 2 Bottom */
    int32_t row, col, future_row, future_col;
    double tour_length;
    uint8_t crossed;
} pf_agent;

/* Byte-identical to pedflow::StepReport (inc/engine.hpp:16-21). */
typedef struct pf_step_report {
    uint32_t step, moved, newly_crossed_top, newly_crossed_bottom;
} pf_step_report;

typedef struct pf_ctx pf_ctx;

/* Ghost/boundary rows of one replica's current planes, for the halo
 * exchange of a row shard. All three are contiguous device ranges. */
typedef struct pf_halo_rows {
    void* cells; size_t cell_bytes; /* PF_GHOST_ROWS rows of u32 cell words */
    void* tau;   size_t tau_bytes;  /* PF_GHOST_ROWS rows of {f64 top, f64 bottom} (ACO) */
    void* tour;  size_t tour_bytes; /* 1 row of f64 tour lengths (ACO) */
    void* occ;   size_t occ_bytes;  /* PF_GHOST_ROWS rows of occupancy bit planes (PF_KERNEL_FUSED; else NULL) */
} pf_halo_rows;

const char* pf_last_error(void);
const char* pf_version(void);

/* validate() (src/config.cpp:101-124) plus the GPU preconditions:
 * W*H < 2^32, 2n < 2^29, shard rows >= PF_GHOST_ROWS. */
int pf_validate(const pf_config* cfg);

/* band_height (src/metrics.cpp:8-11). */
int32_t pf_band_height(int32_t agents_per_side, int32_t width);

/* new_environment (src/state.cpp:54-75) on the host, into caller-owned
 * planes: occ[H*W], index[H*W], agents[2n], tau_top/tau_bot[H*W] (ACO; may
 * be NULL for LEM). */
int pf_new_environment(const pf_config* cfg, uint64_t seed, uint8_t* occ, uint32_t* index, pf_agent* agents,
                       double* tau_top, double* tau_bot);

/* replaces: StepEngine::StepEngine(EngineOptions) (inc/engine.hpp:51). */
int pf_create(const pf_config* cfg, pf_ctx** out);
int pf_destroy(pf_ctx* ctx);

/* Per-replica scenarios. By default replica i runs cfg.seed + i at
 * cfg.agents_per_side (the repeat loop, tools/pedflow.cpp:135). This call
 * overrides either or both per replica (arrays of cfg.replicas entries, NULL
 * keeps the current values), so one context can batch a whole density sweep
 * (tools/pedflow.cpp:159-189): each density is checked as validate() would
 * (src/config.cpp:101-124). Call it before pf_init_environment / pf_load_state;
 * the crossing band (src/metrics.cpp:8-11) follows each replica's density. */
int pf_set_replicas(pf_ctx* ctx, const int32_t* agents_per_side, const uint64_t* seeds);
/* agents_per_side of one replica, or -1 for a bad argument. */
int32_t pf_replica_agents(const pf_ctx* ctx, int32_t replica);

/* new_environment for every replica (its seed and density), built on the host
 * and uploaded; for a shard only the owned rows and ghost rows travel. */
int pf_init_environment(pf_ctx* ctx);

/* Upload / download one replica's SimState (inc/state.hpp:16-31) as the
 * reference's planes over the GLOBAL grid. A shard reads rows
 * [row_begin-3, row_end+3) and writes back only its owned rows (agents living
 * there). n_agents must be 2 * the replica's agents_per_side. */
int pf_load_state(pf_ctx* ctx, int32_t replica, const uint8_t* occ, const uint32_t* index, const pf_agent* agents,
                  uint32_t n_agents, const double* tau_top, const double* tau_bot, uint32_t step);
int pf_store_state(pf_ctx* ctx, int32_t replica, uint8_t* occ, uint32_t* index, pf_agent* agents, uint32_t n_agents,
                   double* tau_top, double* tau_bot, uint32_t* step);

/* replaces: StepEngine::step(SimState&) x n (src/engine.cpp:53-62).
 * Runs n full steps on every replica; out (may be NULL) receives
 * [replicas][n] reports. Synchronous. */
int pf_step(pf_ctx* ctx, uint32_t n, pf_step_report* out);

/* Phase-level stepping, replaces: StepEngine::score_phase / intention_phase /
 * movement_phase / reset_phase (inc/engine.hpp:55-58, src/engine.cpp:64-193).
 * PF_KERNEL_PIPELINE contexts only (the fused kernels run all four phases in
 * one launch). Phases run in order; a full step is SCORE, INTENTION,
 * MOVEMENT, RESET, bit-identical to pf_step. MOVEMENT writes [replicas]
 * reports to out (may be NULL). Between INTENTION and RESET pf_store_state
 * exports the agents' future_row / future_col as the reference has them;
 * pf_store_scores gives the CandidateScores after SCORE (zeros after RESET). */
#define PF_PHASE_SCORE 0
#define PF_PHASE_INTENTION 1
#define PF_PHASE_MOVEMENT 2
#define PF_PHASE_RESET 3
int pf_phase(pf_ctx* ctx, int32_t phase, pf_step_report* out);
/* CandidateScores (lem.hpp:14-17) of one replica by agent id: scores[(id-1)*8 + slot]
 * in goal-relative slot order, owners[id-1] (always the id); either may be NULL. */
int pf_store_scores(pf_ctx* ctx, int32_t replica, double* scores, uint32_t* owners, uint32_t n_agents);
/* Asynchronous variant: enqueue n steps on the context's stream. Reports stay
 * on the device in a ring of the last 1024 steps; pf_read_reports
 * (synchronizes) returns those of steps [step - n, step) as [replicas][n]. */
int pf_step_async(pf_ctx* ctx, uint32_t n);
/* Capture and instantiate (without launching) the CUDA graphs that
 * pf_step_async(n) / pf_step(n) will replay from the current step, so a timed
 * region does not include graph capture. Optional. */
int pf_prepare_steps(pf_ctx* ctx, uint32_t n);
int pf_read_reports(pf_ctx* ctx, pf_step_report* out, uint32_t n);
int pf_synchronize(pf_ctx* ctx);

/* Device-timed step loop: enqueue n steps bracketed by CUDA events on the
 * context stream. *total_ms = step loop; *kernel_ms = mean duration of the
 * dominant (step) kernel measured with per-launch events in a second pass
 * when kernel_ms is non-NULL (state advances by 2n steps in that case). */
int pf_time_steps(pf_ctx* ctx, uint32_t n, float* total_ms, float* kernel_ms);

uint32_t pf_current_step(const pf_ctx* ctx);
void* pf_stream(pf_ctx* ctx); /* cudaStream_t */

/* Count of CUDA kernel launches issued by this context since creation. */
uint64_t pf_launch_count(const pf_ctx* ctx);

/* Halo exchange support for row shards: side 0 = the rows toward row 0,
 * side 1 = toward row H-1; recv 0 = this shard's boundary rows to send,
 * recv 1 = its ghost rows to fill. Valid for the current step parity. */
int pf_halo(pf_ctx* ctx, int32_t replica, int32_t side, int32_t recv, pf_halo_rows* out);

/* Device-to-device halo exchange between two vertically adjacent shards
 * (upper owns the rows just above lower) on the same or peer devices. */
int pf_exchange_pair(pf_ctx* upper, pf_ctx* lower);

/* Page-locked host memory for SimState planes: pf_load_state / pf_store_state
 * DMA such planes directly (pageable planes go through the library's pinned
 * staging buffers with a multi-threaded host copy). NULL on failure. */
void* pf_host_alloc(size_t bytes);
int pf_host_free(void* p);

/* Fused halo exchange (PF_KERNEL_FUSED only): instead of a separate swap
 * after each step, the step kernel stores this shard's PF_GHOST_ROWS boundary
 * rows (planes, arrivals' words and tours, pheromone) straight into the ghost
 * rows of the neighbour shards, through peer memory (NVLink P2P; CUDA IPC
 * between processes). Ordering is per boundary work item inside the kernel:
 * an item touching the ghost rows waits until the neighbour has completed its
 * previous step's boundary items (its stores into our ghost rows are done and
 * it no longer reads the ghost buffers we are about to write), and the last
 * boundary item of a side releases our count into that neighbour's flag.
 * Interior work never waits. No host work or collective per step, so sharded
 * steps batch into CUDA graphs like single-GPU ones. */
typedef struct pf_peer_desc {
    unsigned char ipc[7][64]; /* cudaIpcMemHandle_t of: cell, occ[0], occ[1], tau[0], tau[1], tour, sync flags */
    uint64_t ptr[7];          /* the same allocations as device pointers of the exporting process */
    int32_t device, width, replicas, model, kernel, row_begin, rows_owned, parity;
    uint32_t step, reserved;
    uint64_t plane, occ_plane; /* per-replica elements of the cell / occupancy planes */
} pf_peer_desc;
/* Describe this context for its neighbours (pointers and IPC handles). */
int pf_peer_export(pf_ctx* ctx, pf_peer_desc* out);
/* Link the neighbour on `side` (0: the shard above, ending at row_begin;
 * 1: the shard below). ipc != 0 opens the IPC handles (another process);
 * ipc == 0 uses the pointers (same process, same or peer-capable device).
 * Both shards must be at the same step and parity; link both directions. */
int pf_peer_attach(pf_ctx* ctx, int32_t side, const pf_peer_desc* peer, int32_t ipc);

/* Device-side state audit of one replica, the cell-resident form of
 * check_consistency (src/state.cpp:77-110): every agent cell holds an id in
 * [1, 2n] of the right side, no id twice, no wall inside the arena, and (for
 * an unsharded context) exactly 2n agents. PF_ERR_STATE with the first bad
 * cell otherwise. *agent_cells (may be NULL) = agents found in owned rows.
 * Checks the resident state in place: nothing is downloaded. */
int pf_audit(pf_ctx* ctx, int32_t replica, uint64_t* agent_cells);

/* Device self-test of the keyed generator (src/rng.cpp:43-59,152-156): for
 * n keys computes random_bits, uniform and normal(mu, sigma) ON THE DEVICE
 * (the same device functions the step kernels use). Pins the device RNG and
 * AS241 quantile against the oracle. Outputs may be NULL. */
int pf_selftest_rng(int32_t device, uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                    const uint64_t* entity, const uint32_t* counter, double mu, double sigma, uint64_t* bits_out,
                    double* uniform_out, double* normal_out);

/* Device self-test of the selection functions the step kernels use, over n
 * keys (seed, step, entity): kind 0 lem_select (src/lem.cpp:20-61; scores
 * from d0's distance table, normal(mu_sel*C, sigma_sel*C)), kind 1
 * aco_select (src/aco.cpp:59-93) with caller numerators num[8*i..8*i+7],
 * kind 2 the movement-phase winner draw (src/engine.cpp:116-120) among the
 * row-major contender codes set in mask[i]. mask[i] is the goal-relative
 * open-slot mask (bit 0 = F) for kinds 0/1. out[i] = the chosen slot / code,
 * or -1 (stay / no contender). entity = agent id (0/1) or global cell index (2). */
int pf_selftest_select(int32_t device, int32_t kind, uint32_t n, double d0, double sel_mu, double sel_sigma,
                       const uint8_t* mask, const double* num, const uint64_t* seed, const uint32_t* step,
                       const uint64_t* entity, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
