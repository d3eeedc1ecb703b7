// Internal interface between the C-ABI/context code (pf_context.cu) and the
// kernels (pf_kernels.cu). Not part of the public boundary.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "pf_device.cuh"

namespace pfk {

constexpr int kGhost = 3;  // == PF_GHOST_ROWS

// Device planes of one context. Every plane is replica-major:
// plane[replica][buffer row][column]; buffer row b <-> global row
// row_begin - kGhost + b.
struct Planes {
    // Cell words. PF_KERNEL_FUSED: one plane updated in place (cell[1] ==
    // cell[0]), valid only where occ says "occupied". Other kernels: ping-pong.
    uint32_t* cell[2];
    // PF_KERNEL_FUSED: ping-pong occupancy bit planes, uint2 {v30, v31} per
    // 32-cell segment, rows of wsp segments (2 wall segments of padding on
    // each side: segment s of a row is at index s + 2). Null otherwise.
    uint2* occ[2];
    size_t occ_plane;   // uint2 elements per replica = rows_buf * wsp
    int wsp;
    double2* tau[2];    // ping-pong {top, bottom} pheromone (ACO); float2 data when StepArgs::tau_f32
    double* tour;       // cell-resident tour length, updated in place (ACO)
    uint8_t* intent;    // pipeline-kernel scratch
    uint8_t* win;       // pipeline-kernel scratch
    size_t plane;       // elements per replica plane = rows_buf * W
};

// A neighbouring shard's planes, for the fused halo exchange (PF_KERNEL_FUSED):
// the step kernel mirrors this shard's 3 boundary rows straight into the
// neighbour's ghost rows (peer memory over NVLink, or the same device).
// Buffer row b of this shard is the neighbour's buffer row b + row_delta.
struct PeerRows {
    uint32_t* cell;
    uint2* occ[2];
    double2* tau[2];
    double* tour;
    size_t plane, occ_plane;  // the neighbour's per-replica plane sizes
    int row_delta;
};

struct StepArgs {
    pfdev::StepConsts k;              // by value: hot scalars read from param space
    const pfdev::StepConsts* kc;      // device copy: tables read by the slow paths
    Planes p;
    const pfdev::ReplicaParams* rep;  // [replicas] seed / band / agent count
    const uint32_t* d_step; // device step counter: step of batch slot 0
    uint32_t* reports;      // [replicas][report_cap][4], ring slot = step % report_cap
    int report_cap;
    int row_begin;          // global row of the first owned row
    int rows_owned;
    int rows_buf;           // rows_owned + 2 * kGhost
    int replicas;
    int tiles_per_cta;      // bit kernel: consecutive row tiles per work item (set at launch)
    uint32_t* work;         // bit kernel: work-item counters, one per batch slot (zeroed per batch)
    int num_sms;
    int items_per_cta;      // bit kernel: target work items per resident CTA (load balance vs row reuse)
    PeerRows peer[2];       // [0] the shard above (toward row 0), [1] below; cell == nullptr: none
    int strip_segs;         // bit kernel: 32-column segments per strip (bits_strip_segments)
    int small_tiles;        // bit kernel: -1 auto, 0 / 1 force the small-grid geometry (dev: PEDFLOW_SMALL_TILES)
    // Fused halo ordering (linked shards): sync_local[side] = steps whose
    // boundary items the neighbour on that side has completed (written by it);
    // sync_remote[side] = our flag in the neighbour's memory; bcount = per-step
    // [report_cap][2] completed boundary items per side; err = wait timeout.
    uint32_t* sync_local;
    uint32_t* sync_remote[2];
    uint32_t* bcount;
    uint32_t* err;
    int peer_same_device;   // a linked neighbour shares this GPU: leave it resident slots (no in-kernel wait deadlock)
    // Bit kernel, unlinked contexts: steps per launch (1, or a multi-step
    // launch with tile-level dependencies) and the per-tile completion flags
    // [replicas][strips][tiles] (last completed step + 1; zeroed whenever the
    // step counter is set).
    int nsteps;
    uint32_t* tile_done;
    // ACO pheromone storage: 0 = {f64, f64} per cell (the product), 1 =
    // {f32, f32} (PF_KERNEL_FUSED_F32, tolerance-only); Planes::tau then
    // points at float2 data.
    int tau_f32;
    // LEM: look for windows without agents and skip their S1/S2 (the
    // starting bands of every replica cover < 30% of the rows).
    int skip_empty;
    // LEM, small unlinked grids: CTAs per thread-block cluster of the
    // cluster-resident multi-step kernel (pf_cluster.cu), 0 = not used.
    // Planned once per context (plan_cluster_lem).
    int cluster;
    int cluster_cap;        // its work-list capacity (entries)
    int cluster_nt;         // its threads per CTA (512 or 1024)
};

// Launch one step (batch slot `slot`, reading parity `parity`) on `s`.
// Returns the number of kernel launches issued.
int launch_step_bits(const StepArgs& a, int slot, int parity, cudaStream_t s);   // PF_KERNEL_FUSED
int configure_step_bits();
// Cluster-resident LEM kernel (pf_cluster.cu): the cluster size for these
// args and the largest replica's agent count (0 = not applicable), and a
// launch of a.nsteps steps with it.
int plan_cluster_lem(const StepArgs& a, uint32_t max_agents, int* cap, int* nt);
int launch_cluster_lem(const StepArgs& a, int slot, int parity, cudaStream_t s);
int bits_strip_segments(int width, int model, bool tau_f32);  // strip width in segments (8 or 10)
// Occupancy planes of rows [0, rows) from cell words (W columns; padding
// segments untouched); written to occ0 and, if non-null, occ1.
int launch_build_occ(const uint32_t* words, int W, int rows, int wsp, uint2* occ0, uint2* occ1, cudaStream_t s);
// Zero the words of cells the planes mark empty (stale ids of vacated cells)
// over rows [0, rows); *bad (may be null) += occupied cells whose word's group
// disagrees with the planes.
int launch_sanitize_words(uint32_t* words, const uint2* occ, int W, int rows, int wsp, unsigned long long* bad,
                          cudaStream_t s);
int launch_step_fused(const StepArgs& a, int slot, int parity, cudaStream_t s);  // PF_KERNEL_TILE
int launch_step_pipeline(const StepArgs& a, int slot, int parity, cudaStream_t s);
// *d_step += n
int launch_advance_step(uint32_t* d_step, uint32_t n, cudaStream_t s);
// Fill a tau plane range with {v, v} (f32: float2 elements, v rounded).
int launch_fill_tau(void* p, size_t n, double v, int f32, cudaStream_t s);
int launch_fill_u8(uint8_t* p, size_t n, uint8_t v, cudaStream_t s);
// words[(row - g_lo) * W + col] = (first_id + k) | group << 30 for cells[k] on
// buffer rows [0, rows) (row = cells[k] / W).
int launch_scatter_placement(uint32_t* words, const uint32_t* cells, uint32_t n, uint32_t first_id, uint32_t group,
                             uint32_t W, long long g_lo, int rows, cudaStream_t s);
int launch_audit(const uint32_t* words, size_t first, size_t n, uint32_t n_agents, uint32_t* seen,
                 unsigned long long* counts, cudaStream_t s);
// State upload / download layout transforms.
// (f32: the tau plane holds float2 elements; the reference fields are f64)
int launch_interleave_tau(void* dst, const double* top, const double* bot, size_t n, int f32, cudaStream_t s);
int launch_deinterleave_tau(double* top, double* bot, const void* src, size_t n, int f32, cudaStream_t s);
int launch_gather_tour(double* per_agent, const uint32_t* words, const double* tour, size_t n, cudaStream_t s);
// Reference planes (window rows from g_lo) + AgentRecords -> buffer cell words
// and cell-resident tour; *status = min(buffer cell << 3 | reason) over violations.
int launch_import_state(const uint8_t* occ, const uint32_t* index, const void* agents, uint32_t n_agents, uint32_t W,
                        int H, long long g0, long long g_lo, size_t n, uint32_t* words, double* tour,
                        unsigned long long* status, cudaStream_t s);
// Owned cell words -> reference occupancy / index planes and AgentRecords
// (40-byte pf_agent, by id); status[0] += agent cells, status[1] += bad ids.
// intent (may be null): per-cell intended move codes (between the intention and
// reset phases), exported as the agents' future_row / future_col.
int launch_export_state(const uint32_t* words, const double* tour, const uint8_t* intent, size_t n, uint32_t W,
                        uint32_t row0, uint8_t* occ, uint32_t* index, void* agents, uint32_t n_agents,
                        unsigned long long* status, cudaStream_t s);
// Phase-level stepping (PF_KERNEL_PIPELINE contexts): score_phase into
// scores[replica][n_max][8] / owners[replica][n_max] by agent id; the
// intention phase (propose kernel -> intent plane); the movement phase
// (resolve + commit kernels, counters into the report slot of *d_step).
int launch_score_phase(const StepArgs& a, int parity, double* scores, uint32_t* owners, uint32_t n_max, cudaStream_t s);
int launch_intention_phase(const StepArgs& a, int parity, cudaStream_t s);
int launch_movement_phase(const StepArgs& a, int parity, cudaStream_t s);
int launch_selftest_select(int kind, uint32_t n, const pfdev::StepConsts* kc, const uint8_t* mask, const double* num,
                           const uint64_t* seed, const uint32_t* step, const uint64_t* entity, int32_t* out,
                           cudaStream_t s);
int launch_selftest_rng(uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                        const uint64_t* entity, const uint32_t* counter, double mu, double sigma, uint64_t* bits,
                        double* uni, double* nrm, cudaStream_t s);

}  // namespace pfk
