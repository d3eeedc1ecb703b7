// sm_100a kernels besides the product step kernel (pf_bitstep.cuh):
//
//   step_fused_kernel   PF_KERNEL_TILE cross-check: ONE kernel per step on
//                       ping-pong cell words. A CTA owns a TH x TW tile; it
//                       stages the step-start cell words of the tile plus a
//                       3-cell halo in shared memory, proposes moves for every
//                       agent within 2 cells of the tile, scatters claims into
//                       per-destination bitmasks (shared-memory atomicOr),
//                       resolves every destination within 1 cell (keyed draw
//                       per contested cell), then commits the owned cells.
//   step_pipeline_*     PF_KERNEL_PIPELINE cross-check: the same semantics as
//                       three kernels (propose / resolve / commit) through
//                       global u8 scratch planes.
//   state kernels       SimState import / export / audit, occupancy-plane
//                       build and word sanitising for the product kernel,
//                       pheromone (de)interleave, tour gather.
//   self-tests          the device RNG and selection functions, per key.
//
// Reference semantics: StepEngine::step, src/engine.cpp:53-193.
#include "pf_internal.h"

namespace pfk {

using namespace pfdev;

namespace {

__device__ __forceinline__ void block_count(uint32_t moved, uint32_t ntop, uint32_t nbot, uint32_t* s_cnt,
                                            uint32_t* rep_slot, uint32_t step, bool first_block) {
    moved = __reduce_add_sync(0xFFFFFFFFu, moved);
    ntop = __reduce_add_sync(0xFFFFFFFFu, ntop);
    nbot = __reduce_add_sync(0xFFFFFFFFu, nbot);
    if ((threadIdx.x & 31) == 0 && (moved | ntop | nbot)) {
        if (moved) atomicAdd(&s_cnt[0], moved);
        if (ntop) atomicAdd(&s_cnt[1], ntop);
        if (nbot) atomicAdd(&s_cnt[2], nbot);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (first_block) rep_slot[0] = step;
        if (s_cnt[0]) atomicAdd(&rep_slot[1], s_cnt[0]);
        if (s_cnt[1]) atomicAdd(&rep_slot[2], s_cnt[1]);
        if (s_cnt[2]) atomicAdd(&rep_slot[3], s_cnt[2]);
    }
}

// Commit of one owned cell (the movement-phase commit, src/engine.cpp:137-175,
// plus evaporation src/engine.cpp:124-131 and deposit src/aco.cpp:119-123).
// `w` is the step-start word, `win` the winning source code if the cell was
// empty (kNone otherwise), `vacate` whether the occupant's move was granted,
// `src_word` the winner's word.
template <bool ACO>
__device__ __forceinline__ void commit_cell(const StepConsts& k, int band, uint32_t w, uint8_t win, bool vacate,
                                            uint32_t src_word, int grow, size_t gi, size_t si,
                                            uint32_t* __restrict__ cout, const double2* __restrict__ tin,
                                            double2* __restrict__ tout, double* __restrict__ tour,
                                            uint32_t& moved, uint32_t& ntop, uint32_t& nbot) {
    uint32_t nw = w;
    bool arrived = false;
    uint32_t group = 0;
    double tour_new = 0.0;
    if (w == 0u) {
        if (win != kNone) {
            group = src_word >> 30;
            nw = src_word;
            if (!(src_word & kCrossedBit) && crossed_at(group, grow, k.H, band)) {
                nw |= kCrossedBit;
                if (group == 1u) ++ntop; else ++nbot;
            }
            ++moved;
            arrived = true;
            if (ACO) {
                tour_new = __dadd_rn(tour[si], is_diag(win) ? k.diag : 1.0);
                tour[gi] = tour_new;
            }
        }
    } else if (vacate) {
        nw = 0u;
    }
    cout[gi] = nw;
    if (ACO) {
        double2 t = tin[gi];
        t.x = __dmul_rn(t.x, k.factor);
        t.y = __dmul_rn(t.y, k.factor);
        if (arrived) {
            const double dep = __ddiv_rn(k.q, tour_new);
            if (group == 1u) t.x = __dadd_rn(t.x, dep);
            else t.y = __dadd_rn(t.y, dep);
        }
        tout[gi] = t;
    }
}

}  // namespace

// ------------------------------------------------------------ fused kernel

template <int TH, int TW, bool ACO>
__global__ void __launch_bounds__(256) step_fused_kernel(const StepArgs a, int slot, int parity) {
    constexpr int SH = TH + 6, SW = TW + 6; // staged words: tile + 3-cell halo
    constexpr int RH = TH + 4, RW = TW + 4; // proposal region: tile + 2
    constexpr int CH = TH + 2, CW = TW + 2; // claim/winner region: tile + 1
    __shared__ uint32_t s_cell[SH * SW];
    __shared__ uint32_t s_claim[CH * CW];
    __shared__ uint8_t s_win[CH * CW];
    __shared__ uint8_t s_int[TH * TW];
    __shared__ uint32_t s_cnt[3];

    const StepConsts& k = a.k;
    const int W = k.W;
    const int rep = blockIdx.z;
    const int r0 = blockIdx.y * TH; // owned-local row of the tile origin
    const int c0 = blockIdx.x * TW;
    const uint32_t step = *a.d_step + uint32_t(slot);
    const uint64_t seed = a.rep[rep].seed;
    const size_t base = size_t(rep) * a.p.plane;
    const uint32_t* __restrict__ cin = a.p.cell[parity] + base;
    uint32_t* __restrict__ cout = a.p.cell[parity ^ 1] + base;
    const double2* __restrict__ tin = ACO ? a.p.tau[parity] + base : nullptr;
    double2* __restrict__ tout = ACO ? a.p.tau[parity ^ 1] + base : nullptr;
    double* __restrict__ tour = ACO ? a.p.tour + base : nullptr;

    // Stage the step-start snapshot (walls outside the arena / buffer).
    for (int i = threadIdx.x; i < SH * SW; i += blockDim.x) {
        const int sr = i / SW, sc = i - sr * SW;
        const int b = kGhost + r0 - 3 + sr;
        const int c = c0 - 3 + sc;
        uint32_t w = kWall;
        if (c >= 0 && c < W && b < a.rows_buf) w = __ldg(cin + size_t(b) * W + c);
        s_cell[i] = w;
    }
    for (int i = threadIdx.x; i < CH * CW; i += blockDim.x) s_claim[i] = 0u;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0u;
    __syncthreads();

    // Proposals (score + intention phases) for agents within 2 of the tile;
    // each granted proposal sets bit (7 - code) in its destination's claim mask.
    for (int i = threadIdx.x; i < RH * RW; i += blockDim.x) {
        const int ar = i / RW, ac = i - ar * RW;
        const int sr = ar + 1, sc = ac + 1;
        const uint32_t w = s_cell[sr * SW + sc];
        uint8_t code = kNone;
        if (w != 0u && w != kWall) {
            const int b = kGhost + r0 + ar - 2;
            const int gc = c0 + ac - 2;
            code = propose(
                a.kc, ACO ? 1 : 0, w, seed, step, [&](int dr, int dc) { return s_cell[(sr + dr) * SW + sc + dc]; },
                [&](int dr, int dc, bool bottom) {
                    const double* t = reinterpret_cast<const double*>(tin + size_t(b + dr) * W + (gc + dc));
                    return __ldg(t + (bottom ? 1 : 0));
                });
            if (code != kNone) {
                const int tr = ar - 1 + kDR[code], tc = ac - 1 + kDC[code];
                if (tr >= 0 && tr < CH && tc >= 0 && tc < CW) atomicOr(&s_claim[tr * CW + tc], 1u << (7 - code));
            }
        }
        if (ar >= 2 && ar < TH + 2 && ac >= 2 && ac < TW + 2) s_int[(ar - 2) * TW + (ac - 2)] = code;
    }
    __syncthreads();

    // Cell-centric resolution for destinations within 1 of the tile.
    for (int i = threadIdx.x; i < CH * CW; i += blockDim.x) {
        const uint32_t m = s_claim[i];
        uint8_t wv = kNone;
        if (m) {
            const int cr = i / CW, cc = i - cr * CW;
            const int64_t grow = int64_t(a.row_begin) + r0 + cr - 1;
            wv = resolve(m, seed, step, uint64_t(grow) * uint64_t(W) + uint64_t(c0 + cc - 1));
        }
        s_win[i] = wv;
    }
    __syncthreads();

    // Commit owned cells.
    uint32_t moved = 0, ntop = 0, nbot = 0;
    for (int i = threadIdx.x; i < TH * TW; i += blockDim.x) {
        const int tr = i / TW, tc = i - tr * TW;
        const int lr = r0 + tr, gc = c0 + tc;
        if (lr >= a.rows_owned || gc >= W) continue;
        const int sr = tr + 3, sc = tc + 3;
        const uint32_t w = s_cell[sr * SW + sc];
        const size_t gi = size_t(kGhost + lr) * W + gc;
        uint8_t win = kNone;
        bool vacate = false;
        uint32_t src_word = 0;
        size_t si = 0;
        if (w == 0u) {
            win = s_win[(tr + 1) * CW + tc + 1];
            if (win != kNone) {
                src_word = s_cell[(sr + kDR[win]) * SW + sc + kDC[win]];
                si = size_t(kGhost + lr + kDR[win]) * W + (gc + kDC[win]);
            }
        } else {
            const uint8_t ic = s_int[tr * TW + tc];
            vacate = ic != kNone && s_win[(tr + 1 + kDR[ic]) * CW + tc + 1 + kDC[ic]] == uint8_t(7 - ic);
        }
        commit_cell<ACO>(k, a.rep[rep].band, w, win, vacate, src_word, a.row_begin + lr, gi, si, cout, tin, tout, tour, moved,
                         ntop, nbot);
    }
    uint32_t* rep_slot = a.reports + (size_t(rep) * a.report_cap + step % uint32_t(a.report_cap)) * 4;
    block_count(moved, ntop, nbot, s_cnt, rep_slot, step, blockIdx.x == 0 && blockIdx.y == 0);
}

constexpr int kTH = 32, kTW = 32;

int launch_step_fused(const StepArgs& a, int slot, int parity, cudaStream_t s) {
    dim3 grid((a.k.W + kTW - 1) / kTW, (a.rows_owned + kTH - 1) / kTH, a.replicas);
    if (a.k.model == 1) step_fused_kernel<kTH, kTW, true><<<grid, 256, 0, s>>>(a, slot, parity);
    else step_fused_kernel<kTH, kTW, false><<<grid, 256, 0, s>>>(a, slot, parity);
    return 1;
}

// --------------------------------------------------------- pipeline kernels

// K1: proposals for every agent in buffer rows [kGhost-2, kGhost+rows_owned+2).
__global__ void __launch_bounds__(256) pipeline_propose_kernel(const StepArgs a, int slot, int parity) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = kGhost - 2 + int(blockIdx.y);
    const int rep = blockIdx.z;
    const int W = a.k.W;
    if (c >= W) return;
    const size_t base = size_t(rep) * a.p.plane;
    const uint32_t* cin = a.p.cell[parity] + base;
    const double2* tin = a.k.model == 1 ? a.p.tau[parity] + base : nullptr;
    const uint32_t w = cin[size_t(b) * W + c];
    uint8_t code = kNone;
    if (w != 0u && w != kWall) {
        const uint32_t step = *a.d_step + uint32_t(slot);
        code = propose(
            a.kc, a.k.model, w, a.rep[rep].seed, step,
            [&](int dr, int dc) {
                const int cc = c + dc;
                if (cc < 0 || cc >= W) return kWall;
                return cin[size_t(b + dr) * W + cc];
            },
            [&](int dr, int dc, bool bottom) {
                const double* t = reinterpret_cast<const double*>(tin + size_t(b + dr) * W + (c + dc));
                return t[bottom ? 1 : 0];
            });
    }
    a.p.intent[base + size_t(b) * W + c] = code;
}

// K2: winners for every empty cell in buffer rows [kGhost-1, kGhost+rows_owned+1).
__global__ void __launch_bounds__(256) pipeline_resolve_kernel(const StepArgs a, int slot, int parity) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = kGhost - 1 + int(blockIdx.y);
    const int rep = blockIdx.z;
    const int W = a.k.W;
    if (c >= W) return;
    const size_t base = size_t(rep) * a.p.plane;
    const uint32_t* cin = a.p.cell[parity] + base;
    const uint8_t* intent = a.p.intent + base;
    uint8_t wv = kNone;
    if (cin[size_t(b) * W + c] == 0u) {
        uint32_t claims = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int cc = c + kDC[j];
            if (cc < 0 || cc >= W) continue;
            claims |= uint32_t(intent[size_t(b + kDR[j]) * W + cc] == uint8_t(7 - j)) << j;
        }
        if (claims) {
            const uint32_t step = *a.d_step + uint32_t(slot);
            const int64_t grow = int64_t(a.row_begin) + (b - kGhost);
            wv = resolve(claims, a.rep[rep].seed, step, uint64_t(grow) * uint64_t(W) + uint64_t(c));
        }
    }
    a.p.win[base + size_t(b) * W + c] = wv;
}

// K3: commit owned rows.
template <bool ACO>
__global__ void __launch_bounds__(256) pipeline_commit_kernel(const StepArgs a, int slot, int parity) {
    __shared__ uint32_t s_cnt[3];
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int lr = int(blockIdx.y);
    const int rep = blockIdx.z;
    const int W = a.k.W;
    const size_t base = size_t(rep) * a.p.plane;
    const uint32_t step = *a.d_step + uint32_t(slot);
    uint32_t moved = 0, ntop = 0, nbot = 0;
    if (c < W) {
        const uint32_t* cin = a.p.cell[parity] + base;
        const uint8_t* intent = a.p.intent + base;
        const uint8_t* winp = a.p.win + base;
        const int b = kGhost + lr;
        const size_t gi = size_t(b) * W + c;
        const uint32_t w = cin[gi];
        uint8_t win = kNone;
        bool vacate = false;
        uint32_t src_word = 0;
        size_t si = 0;
        if (w == 0u) {
            win = winp[gi];
            if (win != kNone) {
                si = size_t(b + kDR[win]) * W + (c + kDC[win]);
                src_word = cin[si];
            }
        } else {
            const uint8_t ic = intent[gi];
            vacate = ic != kNone && winp[size_t(b + kDR[ic]) * W + (c + kDC[ic])] == uint8_t(7 - ic);
        }
        commit_cell<ACO>(a.k, a.rep[rep].band, w, win, vacate, src_word, a.row_begin + lr, gi, si, a.p.cell[parity ^ 1] + base,
                         ACO ? a.p.tau[parity] + base : nullptr, ACO ? a.p.tau[parity ^ 1] + base : nullptr,
                         ACO ? a.p.tour + base : nullptr, moved, ntop, nbot);
    }
    uint32_t* rep_slot = a.reports + (size_t(rep) * a.report_cap + step % uint32_t(a.report_cap)) * 4;
    block_count(moved, ntop, nbot, s_cnt, rep_slot, step, blockIdx.x == 0 && blockIdx.y == 0);
}

// score_phase (src/engine.cpp:64-74): every agent's CandidateScores (lem_scores
// src/lem.cpp:8-18 or aco_numerators src/aco.cpp:39-51, goal-relative slot
// order F FL FR L R B BL BR) by agent id; the values the selection uses.
__global__ void __launch_bounds__(256) score_kernel(const StepArgs a, int parity, double* scores, uint32_t* owners,
                                                    uint32_t n_max) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = kGhost + int(blockIdx.y);
    const int rep = blockIdx.z;
    const int W = a.k.W;
    if (c >= W) return;
    const size_t base = size_t(rep) * a.p.plane;
    const uint32_t* cin = a.p.cell[parity] + base;
    const uint32_t w = cin[size_t(b) * W + c];
    if (w == 0u || w == kWall) return;
    const uint32_t id = w & kIdMask;
    if (id == 0u || id > n_max) return;
    const bool bottom = (w >> 30) == 2u;
    const double2* tin = a.k.model == 1 ? a.p.tau[parity] + base : nullptr;
    double* out = scores + (size_t(rep) * n_max + (id - 1)) * 8;
    for (int i = 0; i < 8; ++i) {
        const uint8_t code = bottom ? uint8_t(7 - kSlotCodeTop[i]) : kSlotCodeTop[i];
        const int cc = c + kDC[code];
        const bool open = cc >= 0 && cc < W && cin[size_t(b + kDR[code]) * W + cc] == 0u;
        double v = 0.0;
        if (open) {
            if (a.k.model == 0) {
                v = a.kc->lem_score[i];
            } else {
                const double* t = reinterpret_cast<const double*>(tin + size_t(b + kDR[code]) * W + cc);
                v = __dmul_rn(pheromone_term(a.kc, t[bottom ? 1 : 0]), a.kc->eta[i]);
            }
        }
        out[i] = v;
    }
    if (owners) owners[size_t(rep) * n_max + (id - 1)] = id;
}

int launch_score_phase(const StepArgs& a, int parity, double* scores, uint32_t* owners, uint32_t n_max, cudaStream_t s) {
    score_kernel<<<dim3((a.k.W + 255) / 256, a.rows_owned, a.replicas), 256, 0, s>>>(a, parity, scores, owners, n_max);
    return 1;
}

int launch_intention_phase(const StepArgs& a, int parity, cudaStream_t s) {
    pipeline_propose_kernel<<<dim3((a.k.W + 255) / 256, a.rows_owned + 4, a.replicas), 256, 0, s>>>(a, 0, parity);
    return 1;
}

int launch_movement_phase(const StepArgs& a, int parity, cudaStream_t s) {
    const int bx = (a.k.W + 255) / 256;
    pipeline_resolve_kernel<<<dim3(bx, a.rows_owned + 2, a.replicas), 256, 0, s>>>(a, 0, parity);
    if (a.k.model == 1) pipeline_commit_kernel<true><<<dim3(bx, a.rows_owned, a.replicas), 256, 0, s>>>(a, 0, parity);
    else pipeline_commit_kernel<false><<<dim3(bx, a.rows_owned, a.replicas), 256, 0, s>>>(a, 0, parity);
    return 2;
}

int launch_step_pipeline(const StepArgs& a, int slot, int parity, cudaStream_t s) {
    const int bx = (a.k.W + 255) / 256;
    pipeline_propose_kernel<<<dim3(bx, a.rows_owned + 4, a.replicas), 256, 0, s>>>(a, slot, parity);
    pipeline_resolve_kernel<<<dim3(bx, a.rows_owned + 2, a.replicas), 256, 0, s>>>(a, slot, parity);
    if (a.k.model == 1) pipeline_commit_kernel<true><<<dim3(bx, a.rows_owned, a.replicas), 256, 0, s>>>(a, slot, parity);
    else pipeline_commit_kernel<false><<<dim3(bx, a.rows_owned, a.replicas), 256, 0, s>>>(a, slot, parity);
    return 3;
}

// ----------------------------------------------------------------- helpers

__global__ void advance_step_kernel(uint32_t* d_step, uint32_t n) { *d_step += n; }

int launch_advance_step(uint32_t* d_step, uint32_t n, cudaStream_t s) {
    advance_step_kernel<<<1, 1, 0, s>>>(d_step, n);
    return 1;
}

__global__ void fill_tau_kernel(double2* p, size_t n, double v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = make_double2(v, v);
}
__global__ void fill_tau_f32_kernel(float2* p, size_t n, float v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = make_float2(v, v);
}

int launch_fill_tau(void* p, size_t n, double v, int f32, cudaStream_t s) {
    if (f32) fill_tau_f32_kernel<<<148 * 8, 256, 0, s>>>(static_cast<float2*>(p), n, static_cast<float>(v));
    else fill_tau_kernel<<<148 * 8, 256, 0, s>>>(static_cast<double2*>(p), n, v);
    return 1;
}

// new_environment on the device: the placed agents' cell words
// (id | group << 30, src/state.cpp:38-48) scattered into the buffer rows
// [g_lo, g_lo + rows) of a zeroed word plane. cells[k] = global linear cell of
// agent first_id + k (the host's keyed Fisher-Yates, pf_setup.cpp).
__global__ void scatter_placement_kernel(uint32_t* words, const uint32_t* cells, uint32_t n, uint32_t first_id,
                                         uint32_t group, uint32_t W, long long g_lo, int rows) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t cell = cells[k];
        const long long row = (long long)(cell / W) - g_lo;
        if (row >= 0 && row < rows) words[size_t(row) * W + cell % W] = (first_id + k) | (group << 30);
    }
}

int launch_scatter_placement(uint32_t* words, const uint32_t* cells, uint32_t n, uint32_t first_id, uint32_t group,
                             uint32_t W, long long g_lo, int rows, cudaStream_t s) {
    if (n == 0) return 0;
    scatter_placement_kernel<<<148 * 8, 256, 0, s>>>(words, cells, n, first_id, group, W, g_lo, rows);
    return 1;
}

__global__ void fill_u8_kernel(uint8_t* p, size_t n, uint8_t v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

int launch_fill_u8(uint8_t* p, size_t n, uint8_t v, cudaStream_t s) {
    fill_u8_kernel<<<148 * 8, 256, 0, s>>>(p, n, v);
    return 1;
}

// --- state upload / download layout transforms (pf_load_state / pf_store_state)

__global__ void interleave_tau_kernel(double2* dst, const double* top, const double* bot, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = make_double2(top[i], bot[i]);
}
__global__ void interleave_tau_f32_kernel(float2* dst, const double* top, const double* bot, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = make_float2(__double2float_rn(top[i]), __double2float_rn(bot[i]));
}

__global__ void deinterleave_tau_kernel(double* top, double* bot, const double2* src, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const double2 t = src[i];
        top[i] = t.x;
        bot[i] = t.y;
    }
}
__global__ void deinterleave_tau_f32_kernel(double* top, double* bot, const float2* src, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const float2 t = src[i];
        top[i] = double(t.x);
        bot[i] = double(t.y);
    }
}

// per_agent[id - 1] = tour[cell] for agent cells.
__global__ void gather_tour_kernel(double* per_agent, const uint32_t* words, const double* tour, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = words[i];
        if (w != 0u && w != pfdev::kWall) per_agent[(w & pfdev::kIdMask) - 1] = tour[i];
    }
}

// State import: the check_consistency-style audit (src/state.cpp:77-110) of
// the uploaded reference planes and their conversion to cell words, per
// buffer cell. Buffer row b is global row g0 + b; rows outside the grid are
// walls; occ/index hold the window rows from g_lo. Agent records are the
// 40-byte pf_agent as five u64 words (see export_state_kernel). The first
// violating buffer cell is reported as status = min(cell << 3 | reason), with
// the reasons of pf_load_state.
__global__ void import_state_kernel(const uint8_t* __restrict__ occ, const uint32_t* __restrict__ index,
                                    const unsigned long long* __restrict__ agents, uint32_t n_agents, uint32_t W,
                                    int H, long long g0, long long g_lo, size_t n, uint32_t* __restrict__ words,
                                    double* __restrict__ tour, unsigned long long* status) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const long long g = g0 + (long long)(i / W);
        const uint32_t col = uint32_t(i % W);
        uint32_t w = pfdev::kWall;
        double t = 0.0;
        unsigned why = 0;
        if (g >= 0 && g < H) {
            const size_t wi = size_t(g - g_lo) * W + col;
            const uint32_t id = index[wi];
            const uint32_t o = occ[wi];
            w = 0u;
            if ((id == 0u) != (o == 0u)) why = 1;
            else if (id != 0u) {
                if (id > n_agents) why = 2;
                else {
                    const unsigned long long* a = agents + size_t(id - 1) * 5;
                    const unsigned long long q0 = a[0], q1 = a[1];
                    const uint32_t grp = uint32_t(q0 >> 32) & 0xFFu;
                    if (uint32_t(q0) != id) why = 3;
                    else if (int32_t(uint32_t(q1)) != g || int32_t(uint32_t(q1 >> 32)) != int32_t(col)) why = 4;
                    else if (grp != o || (grp != 1u && grp != 2u)) why = 5;
                    else {
                        w = id | ((a[4] & 0xFFull) ? pfdev::kCrossedBit : 0u) | (grp << 30);
                        t = __longlong_as_double(static_cast<long long>(a[3]));
                    }
                }
            }
        }
        if (why) {
            atomicMin(status, (static_cast<unsigned long long>(i) << 3) | why);
            w = 0u;
        }
        words[i] = w;
        if (tour) tour[i] = t;
    }
}

// Whole-grid export into the reference's SimState planes (the inverse of the
// host conversion in pf_load_state): per owned cell, occupancy (u8) and index
// (u32) in row-major order, and for an agent cell its AgentRecord
// (inc/grid.hpp:84-93, 40 bytes as five u64 words: index | group << 32,
// row | col << 32, future_row | future_col << 32 (= position after the
// reset phase, src/engine.cpp:183-193), tour_length, crossed; padding zero).
// status[0] += agent cells, status[1] += cells with an out-of-range id.
__global__ void export_state_kernel(const uint32_t* __restrict__ words, const double* __restrict__ tour,
                                    const uint8_t* __restrict__ intent, size_t n, uint32_t W, uint32_t row0,
                                    uint8_t* __restrict__ occ, uint32_t* __restrict__ index,
                                    unsigned long long* __restrict__ agents, uint32_t n_agents,
                                    unsigned long long* status) {
    unsigned long long found = 0, bad = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = words[i];
        const uint32_t id = w & pfdev::kIdMask;
        if (occ) occ[i] = uint8_t(w ? (w >> 30) : 0u);
        if (index) index[i] = w ? id : 0u;
        if (!w) continue;
        if (id == 0u || id > n_agents) {
            ++bad;
            continue;
        }
        ++found;
        if (agents) {
            const unsigned long long row = uint32_t(row0 + uint32_t(i / W)), col = uint32_t(i % W);
            unsigned long long* a = agents + size_t(id - 1) * 5;
            a[0] = id | (static_cast<unsigned long long>(w >> 30) << 32);
            a[1] = row | (col << 32);
            // Between intention_phase and reset_phase the future is the intended
            // cell (a mover's is its new cell: it arrived where no intent was).
            const uint8_t code = intent ? intent[i] : pfdev::kNone;
            if (code == pfdev::kNone) {
                a[2] = row | (col << 32);
            } else {
                const unsigned long long fr = uint32_t(int(row) + pfdev::kDR[code]);
                const unsigned long long fc = uint32_t(int(col) + pfdev::kDC[code]);
                a[2] = fr | (fc << 32);
            }
            a[3] = tour ? static_cast<unsigned long long>(__double_as_longlong(tour[i])) : 0ull;
            a[4] = (w & pfdev::kCrossedBit) ? 1ull : 0ull;
        }
    }
    for (int o = 16; o; o >>= 1) {
        found += __shfl_xor_sync(0xFFFFFFFFu, found, o);
        bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (found) atomicAdd(&status[0], found);
        if (bad) atomicAdd(&status[1], bad);
    }
}

// Device-side state audit (check_consistency, src/state.cpp:77-110, in the
// cell-resident layout): every agent cell holds an id in [1, n_agents] whose
// group matches its side (ids 1..n Top, n+1..2n Bottom, src/state.cpp:72-73),
// no id appears twice (bitmap), no wall inside the arena. counts[0] = agent
// cells, counts[1] = violations, counts[2] = first violating cell + 1.
__global__ void audit_kernel(const uint32_t* words, size_t first, size_t n, uint32_t n_agents, uint32_t* seen,
                             unsigned long long* counts) {
    unsigned long long agents = 0;
    for (size_t i = first + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < first + n;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = words[i];
        if (w == 0u) continue;
        bool bad = w == pfdev::kWall;
        if (!bad) {
            const uint32_t id = w & pfdev::kIdMask, g = w >> 30;
            bad = id == 0u || id > n_agents || g != (id <= n_agents / 2 ? 1u : 2u);
            if (!bad) {
                const uint32_t b = 1u << ((id - 1) & 31u);
                bad = (atomicOr(&seen[(id - 1) >> 5], b) & b) != 0u;  // duplicate id
                ++agents;
            }
        }
        if (bad) {
            atomicAdd(&counts[1], 1ull);
            atomicMin(&counts[2], (unsigned long long)(i - first + 1));
        }
    }
    agents = __reduce_add_sync(0xFFFFFFFFu, unsigned(agents));
    if ((threadIdx.x & 31) == 0 && agents) atomicAdd(&counts[0], agents);
}

int launch_audit(const uint32_t* words, size_t first, size_t n, uint32_t n_agents, uint32_t* seen,
                 unsigned long long* counts, cudaStream_t s) {
    audit_kernel<<<148 * 8, 256, 0, s>>>(words, first, n, n_agents, seen, counts);
    return 1;
}

int launch_interleave_tau(void* dst, const double* top, const double* bot, size_t n, int f32, cudaStream_t s) {
    if (f32) interleave_tau_f32_kernel<<<148 * 8, 256, 0, s>>>(static_cast<float2*>(dst), top, bot, n);
    else interleave_tau_kernel<<<148 * 8, 256, 0, s>>>(static_cast<double2*>(dst), top, bot, n);
    return 1;
}
int launch_deinterleave_tau(double* top, double* bot, const void* src, size_t n, int f32, cudaStream_t s) {
    if (f32) deinterleave_tau_f32_kernel<<<148 * 8, 256, 0, s>>>(top, bot, static_cast<const float2*>(src), n);
    else deinterleave_tau_kernel<<<148 * 8, 256, 0, s>>>(top, bot, static_cast<const double2*>(src), n);
    return 1;
}
int launch_import_state(const uint8_t* occ, const uint32_t* index, const void* agents, uint32_t n_agents, uint32_t W,
                        int H, long long g0, long long g_lo, size_t n, uint32_t* words, double* tour,
                        unsigned long long* status, cudaStream_t s) {
    import_state_kernel<<<148 * 8, 256, 0, s>>>(occ, index, static_cast<const unsigned long long*>(agents), n_agents,
                                                W, H, g0, g_lo, n, words, tour, status);
    return 1;
}
int launch_export_state(const uint32_t* words, const double* tour, const uint8_t* intent, size_t n, uint32_t W,
                        uint32_t row0, uint8_t* occ, uint32_t* index, void* agents, uint32_t n_agents,
                        unsigned long long* status, cudaStream_t s) {
    export_state_kernel<<<148 * 8, 256, 0, s>>>(words, tour, intent, n, W, row0, occ, index,
                                                static_cast<unsigned long long*>(agents), n_agents, status);
    return 1;
}
int launch_gather_tour(double* per_agent, const uint32_t* words, const double* tour, size_t n, cudaStream_t s) {
    gather_tour_kernel<<<148 * 8, 256, 0, s>>>(per_agent, words, tour, n);
    return 1;
}

// --- occupancy bit planes of the fused kernel (pf_bitstep.cuh) ----------

// Warp per 32-cell segment, lane = column: two ballots of the word's group
// bits; columns past W are walls (both bits set).
__global__ void build_occ_kernel(const uint32_t* __restrict__ words, int W, int rows, int wsp, uint2* occ0,
                                 uint2* occ1) {
    const int lane = threadIdx.x & 31;
    const int nseg = (W + 31) / 32;
    const size_t units = size_t(rows) * nseg;
    for (size_t u = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) / 32; u < units;
         u += size_t(gridDim.x) * blockDim.x / 32) {
        const size_t row = u / nseg;
        const int seg = int(u % nseg), c = 32 * seg + lane;
        const uint32_t w = c < W ? words[row * W + c] : pfdev::kWall;
        const uint2 p = make_uint2(__ballot_sync(0xFFFFFFFFu, (w >> 30) & 1u), __ballot_sync(0xFFFFFFFFu, w >> 31));
        if (lane == 0) {
            occ0[row * wsp + seg + 2] = p;
            if (occ1) occ1[row * wsp + seg + 2] = p;
        }
    }
}

int launch_build_occ(const uint32_t* words, int W, int rows, int wsp, uint2* occ0, uint2* occ1, cudaStream_t s) {
    build_occ_kernel<<<148 * 8, 256, 0, s>>>(words, W, rows, wsp, occ0, occ1);
    return 1;
}

// Thread per cell: a word under an empty plane bit is a stale id of a
// vacated cell (the fused kernel never clears them) and becomes 0.
__global__ void sanitize_words_kernel(uint32_t* words, const uint2* __restrict__ occ, int W, int rows, int wsp,
                                      unsigned long long* bad) {
    const size_t n = size_t(rows) * W;
    unsigned nbad = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const size_t row = i / W;
        const int c = int(i - row * W);
        const uint2 p = occ[row * wsp + c / 32 + 2];
        const uint32_t g = ((p.x >> (c & 31)) & 1u) | ((p.y >> (c & 31)) & 1u) << 1;
        const uint32_t w = words[i];
        if (g == 0u) {
            if (w != 0u) words[i] = 0u;
        } else if ((w >> 30) != g || (g != 3u && (w & pfdev::kIdMask) == 0u)) {
            ++nbad;
        }
    }
    if (bad) {
        nbad = __reduce_add_sync(0xFFFFFFFFu, nbad);
        if ((threadIdx.x & 31) == 0 && nbad) atomicAdd(bad, (unsigned long long)nbad);
    }
}

int launch_sanitize_words(uint32_t* words, const uint2* occ, int W, int rows, int wsp, unsigned long long* bad,
                          cudaStream_t s) {
    sanitize_words_kernel<<<148 * 8, 256, 0, s>>>(words, occ, W, rows, wsp, bad);
    return 1;
}

}  // namespace pfk

namespace pfk {

__global__ void selftest_rng_kernel(uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                                    const uint64_t* entity, const uint32_t* counter, double mu, double sigma,
                                    uint64_t* bits, double* uni, double* nrm) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t b = pfdev::philox_bits(seed[i], step[i], phase[i], entity[i], counter[i]);
    bits[i] = b;
    uni[i] = pfdev::uniform_from_bits(b);
    const double u = __dmul_rn(__dadd_rn(__ull2double_rn(b >> 11), 0.5), 0x1.0p-53);
    nrm[i] = __dadd_rn(mu, __dmul_rn(sigma, pfdev::inverse_normal_cdf(u)));
}

// Selection self-test (pf_selftest_select): the device's lem_select /
// aco_select (forward priority + lem_choose / aco_choose) and the cell-centric
// resolve, exactly as the step kernels call them, over arrays of keys.
__global__ void selftest_select_kernel(int kind, uint32_t n, const pfdev::StepConsts* kc, const uint8_t* mask,
                                       const double* num, const uint64_t* seed, const uint32_t* step,
                                       const uint64_t* entity, int32_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t m = mask[i];
    int r;
    if (kind == 2) {
        r = m ? int(pfdev::resolve(m, seed[i], step[i], entity[i])) : -1;
    } else if (m & 1u) {
        r = 0;  // forward open: move forward, no draw (src/lem.cpp:23-26, src/aco.cpp:60-63)
    } else if (m == 0u) {
        r = -1;  // boxed in: stay
    } else if (kind == 0) {
        r = pfdev::lem_choose(kc, m, seed[i], step[i], uint32_t(entity[i]));
    } else {
        double v[8];
        for (int k = 0; k < 8; ++k) v[k] = num[size_t(i) * 8 + k];
        r = pfdev::aco_choose(v, m, seed[i], step[i], uint32_t(entity[i]));
    }
    out[i] = r;
}

int launch_selftest_select(int kind, uint32_t n, const pfdev::StepConsts* kc, const uint8_t* mask, const double* num,
                           const uint64_t* seed, const uint32_t* step, const uint64_t* entity, int32_t* out,
                           cudaStream_t s) {
    selftest_select_kernel<<<(n + 255) / 256, 256, 0, s>>>(kind, n, kc, mask, num, seed, step, entity, out);
    return 1;
}

int launch_selftest_rng(uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                        const uint64_t* entity, const uint32_t* counter, double mu, double sigma, uint64_t* bits,
                        double* uni, double* nrm, cudaStream_t s) {
    selftest_rng_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, seed, step, phase, entity, counter, mu, sigma, bits, uni,
                                                         nrm);
    return 1;
}

}  // namespace pfk
