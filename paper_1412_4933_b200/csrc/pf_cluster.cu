// Cluster-resident multi-step kernel for small sparse LEM scenarios (single
// 480^2 runs such as C1; PF_KERNEL_FUSED).
//
// A single small scenario is latency-bound on the persistent bit-plane kernel
// (pf_bitstep.cuh): every step is a dependent chain of launch, TMA window
// load from L2, three CTA barriers and a flush, ~5 us even on an empty grid.
// Here one thread-block cluster (16 CTAs, one per SM, non-portable size; 8
// where 16 cannot be co-scheduled) holds the whole replica in shared memory
// for all the steps of a launch: the grid is loaded once, every step runs
// on-chip between two cluster barriers, and the result is written back once.
// A LEM cell is its 32-bit word (id | crossed | group, 0 = empty) plus one
// claim byte. Only sparse grids take this path (kMaxDensity): 16 SMs issue
// every proposal, so dense grids keep the whole GPU.
//
// Layout: CTA q of a replica's cluster owns the column slice
// [q * cpc, (q + 1) * cpc) of every row, so the crowds' horizontal bands
// spread evenly over the CTAs. Its words are held with one ghost column on
// each side (copies of the neighbours' edge columns, kWall at the arena's
// edges) and a wall row above and below, so every proposal reads local
// shared memory only. The work of a step is listed, not scanned: the slice's
// agents (u16 entries row << cb | column) and its claimed cells. Sparse
// replica batches run one cluster per replica, in waves.
//
// One step (StepEngine::step, src/engine.cpp:53-193):
//   S1  per listed agent: the LEM proposal (score_phase + intention_phase,
//       src/engine.cpp:64-90, src/lem.cpp:20-60: the same forward priority
//       and lem_choose_with as the other kernels, its tables in shared
//       memory); a proposing agent ORs its claim bit (the row-major code of
//       its cell seen from the destination) into the destination's claim
//       byte, local or in a neighbour's slice (DSMEM atomics; OR commutes, so
//       the result is order-independent), and the first claimer of a cell
//       lists it with the cell's owner.
//   --- cluster barrier
//   S2  per listed claimed cell (empty at step start by construction): the
//       keyed resolution on the global cell index (src/engine.cpp:101-122,
//       pfdev::resolve), then the commit (src/engine.cpp:137-175): the
//       winner's word moves in (crossed bit and counters, src/metrics.cpp:13-16)
//       and its source is cleared, with the ghost copies (DSMEM stores). Each
//       source is read and cleared only by the one destination it won, and
//       destinations were empty at step start, so no two threads touch the
//       same word.
//   --- cluster barrier
// Counters go to the report ring once per launch.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "pf_internal.h"

namespace cg = cooperative_groups;

namespace pfk {
namespace cluster_lem {

using namespace pfdev;

// Threads per CTA: 512 when a CTA's slice holds at most one agent per thread
// on average (C1: 128), else 1,024 (kernel template parameter; picked in
// plan_cluster_lem). A/B on C1: 512 threads 2.2 / 4.1 us per step before /
// after the crowds meet, 1,024 threads 2.5 / 4.4 us (fewer idle warps at the
// cluster barriers); at 10,240 agents per side 1,024 threads are 5% faster.
constexpr size_t kSmemMax = 227 * 1024 - 4096;  // dynamic shared memory per CTA (static: counters, tables)
constexpr int kMaxSteps = 256;                  // steps per launch (the context's graph batch)
// Shorter launches take the bit-plane kernel: loading and writing back the
// replica costs ~24 us per launch (C1 one step per launch: 27 us against
// 8.2 us on the bit-plane kernel), so the cluster kernel pays from ~5 steps on.
constexpr int kMinSteps = 8;
// Replica batches (one cluster per replica, in waves when they outnumber the
// resident clusters): C1 x64 (0.9% density, clusters in waves)
// 23.4 -> 16.4 us/step; denser batches keep the bit-plane kernel.
constexpr long long kMaxWaves = 8;
constexpr double kMaxDensityBatch = 0.02;
constexpr double kMaxDensity = 0.10;            // agents per cell (tools/cluster_sweep.py: faster up to ~12%)

struct Geometry {
    int cl;   // CTAs per cluster (one replica per cluster)
    int cpc;  // columns per CTA
    int cb;   // list-entry column bits
    int cap;  // entries per work list: min(2 x agents of the largest replica, cells per slice)
    size_t bytes;
};

// Words: (H + 2) rows of cpc + 2 columns; claims: H rows of cpc rounded up
// to whole u32 words (4 cells each); then three u16 work lists of cap entries
// (agents at step start, twice for ping-pong, and claimed cells).
__host__ __device__ inline int word_pitch(int cpc) { return cpc + 2; }
__host__ __device__ inline int claim_pitch(int cpc) { return (cpc + 3) / 4 * 4; }
__host__ __device__ inline size_t words_bytes(int H, int cpc) {
    return (size_t(H + 2) * word_pitch(cpc) * 4 + 15) / 16 * 16;
}
__host__ __device__ inline size_t claims_bytes(int H, int cpc) { return size_t(H) * claim_pitch(cpc); }
__host__ __device__ inline size_t smem_bytes(int H, int cpc, int cap) {
    return words_bytes(H, cpc) + claims_bytes(H, cpc) + 3 * size_t(cap) * 2;
}

// List entry (u16): row << cb | slice column, cb = the column bits of the
// slice width (geometry()).

// kDR / kDC / kSlotCodeTop as immediates (lanes index them divergently; the
// constant bank would serialise the distinct addresses).
__device__ __forceinline__ int dr_of(int c) { return int((0xA940u >> (2 * c)) & 3u) - 1; }
__device__ __forceinline__ int dc_of(int c) { return int((0x9224u >> (2 * c)) & 3u) - 1; }
__device__ __forceinline__ int slot_code(int slot, bool bottom) {
    const int c = int((0x40C7EEu >> (3 * slot)) & 7u);
    return bottom ? 7 - c : c;
}

// Append the calling lanes' entries (pred) to a shared-memory list of cap
// entries: one counter atomic per warp. Every lane of the warp must call it.
// The capacities are proven bounds (geometry()); an overflow would be an
// internal error: it is not written and sets bit 2 of *err.
__device__ __forceinline__ void append(uint16_t* list, uint32_t* count, bool pred, uint16_t e, uint32_t cap,
                                       uint32_t* err) {
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, pred);
    if (m == 0u) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, uint32_t(__popc(m)));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    const uint32_t i = base + __popc(m & ((1u << lane) - 1u));
    if (pred && i < cap) list[i] = e;
    if (pred && i >= cap) atomicOr(err, 4u);
}

// glibc's log table (the AS241 tail) and the LEM constants in shared memory:
// global loads after a cluster barrier (which invalidates L1) would each be
// an L2 round trip.
struct SharedLogTab {
    const double* t;  // kLogTab row-major, then kLogPoly
    __device__ double tab(int i, int j) const { return t[2 * i + j]; }
    __device__ double poly(int i) const { return t[256 + i]; }
};
struct SharedLemTab {
    static constexpr bool kEagerTie = true;  // (the draw chain is this kernel's critical path)
    const double* tab;
    const double* logt;
    double m, sg;
    __device__ double score(int i) const { return tab[i]; }
    __device__ double mu() const { return m; }
    __device__ double sigma() const { return sg; }
    // Inlined here (the other kernels call it out of line): no call/return and
    // register save around it on the draw chain (jammed C1 4.05 -> 3.94 us).
    __device__ double normal(double u) const { return inverse_normal_cdf_with(SharedLogTab{logt}, u); }
};

template <int NT>
__global__ void __launch_bounds__(NT, 1) lem_cluster_kernel(const StepArgs a, int slot_idx, int parity, int cpc,
                                                            int cap, int cb) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t cnt[kMaxSteps][3];       // per-step counters, flushed once at the end
    __shared__ uint32_t nagents[2], nclaims[2];  // list lengths, by step parity
    __shared__ double score_tab[8];
    __shared__ double log_tab[2 * 128 + 5];
    cg::cluster_group cluster = cg::this_cluster();
    const int q = int(cluster.block_rank()), cl = int(cluster.num_blocks());
    const int rep = int(blockIdx.x) / cl;
    const int W = a.k.W, H = a.rows_owned;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c_lo = q * cpc, ncols = max(0, min(W, c_lo + cpc) - c_lo);
    const int P = word_pitch(cpc), CP = claim_pitch(cpc);
    uint32_t* const word = reinterpret_cast<uint32_t*>(smem);
    uint8_t* const claim8 = smem + words_bytes(H, cpc);
    uint32_t* const claim32 = reinterpret_cast<uint32_t*>(claim8);
    uint16_t* const agents0 = reinterpret_cast<uint16_t*>(claim8 + claims_bytes(H, cpc));
    uint16_t* const claimed = agents0 + 2 * size_t(cap);
    auto entry = [cb](int r, int lc) { return uint16_t(r << cb | lc); };
    auto entry_row = [cb](uint32_t e) { return int(e >> cb); };
    auto entry_col = [cb](uint32_t e) { return int(e & ((1u << cb) - 1u)); };
    // Word (r, lc), r in -1 .. H, lc in -1 .. cpc.
    auto at = [P](int r, int lc) { return (r + 1) * P + (lc + 1); };
    // The neighbours' arrays (same geometry).
    uint32_t* const word_l = q > 0 ? cluster.map_shared_rank(word, q - 1) : nullptr;
    uint32_t* const word_r = q + 1 < cl ? cluster.map_shared_rank(word, q + 1) : nullptr;
    uint32_t* const claim_l = q > 0 ? cluster.map_shared_rank(claim32, q - 1) : nullptr;
    uint32_t* const claim_r = q + 1 < cl ? cluster.map_shared_rank(claim32, q + 1) : nullptr;
    uint16_t* const claimed_l = q > 0 ? cluster.map_shared_rank(claimed, q - 1) : nullptr;
    uint16_t* const claimed_r = q + 1 < cl ? cluster.map_shared_rank(claimed, q + 1) : nullptr;
    uint32_t* const nclaims_l = q > 0 ? cluster.map_shared_rank(&nclaims[0], q - 1) : nullptr;
    uint32_t* const nclaims_r = q + 1 < cl ? cluster.map_shared_rank(&nclaims[0], q + 1) : nullptr;

    for (int i = threadIdx.x; i < 3 * kMaxSteps; i += NT) (&cnt[0][0])[i] = 0u;
    if (threadIdx.x < 2) nagents[threadIdx.x] = nclaims[threadIdx.x] = 0u;
    if (threadIdx.x < 8) score_tab[threadIdx.x] = a.k.lem_score[threadIdx.x];
    if (threadIdx.x < 256) log_tab[threadIdx.x] = kLogTab[threadIdx.x >> 1][threadIdx.x & 1];
    if (threadIdx.x < 5) log_tab[256 + threadIdx.x] = kLogPoly[threadIdx.x];
    for (int i = threadIdx.x; i < H * CP / 4; i += NT) claim32[i] = 0u;
    for (int i = threadIdx.x; i < P; i += NT) {  // wall rows
        word[at(-1, i - 1)] = kWall;
        word[at(H, i - 1)] = kWall;
    }
    __syncthreads();  // counters
    // Launched with programmatic stream serialization: from here on the
    // previous launch's planes, words and step counter are complete.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t step0 = *a.d_step + uint32_t(slot_idx);
    const uint64_t seed = __ldg(&a.rep[rep].seed);
    const int band = __ldg(&a.rep[rep].band);
    uint32_t* const cw = a.p.cell[0] + size_t(rep) * a.p.plane;
    const uint2* const occ_in = a.p.occ[parity] + size_t(rep) * a.p.occ_plane;
    const int wsp = a.p.wsp;
    // Load the slice and its ghost columns (a word counts only where the
    // step-start planes say occupied; outside the arena and past the last
    // slice's columns: kWall), and list the slice's agents.
    for (int r = warp; r < H; r += NW) {
        const size_t b = size_t(kGhost + r);
        for (int lc0 = -1; lc0 <= cpc; lc0 += 32) {
            const int lc = lc0 + lane, c = c_lo + lc;
            uint32_t w = kWall;
            if (lc <= cpc && c >= 0 && c < W && (lc < ncols || lc == cpc)) {
                const uint2 p = occ_in[b * wsp + (c >> 5) + 2];
                w = (((p.x | p.y) >> (c & 31)) & 1u) ? cw[b * W + c] : 0u;
            }
            if (lc <= cpc) word[at(r, lc)] = w;
            append(agents0, &nagents[0], lc >= 0 && lc < ncols && w != 0u, entry(r, lc), cap, a.err);
        }
    }
    cluster.sync();

    const SharedLemTab tab{score_tab, log_tab, a.k.sel_mu, a.k.sel_sigma};
    const int n = a.nsteps;
    uint32_t moved = 0, ntop = 0, nbot = 0;
    for (int s = 0; s < n; ++s) {
        const uint32_t step = step0 + uint32_t(s);
        const int cur = s & 1;
        const uint16_t* const agents_in = agents0 + size_t(cur) * cap;
        uint16_t* const agents_out = agents0 + size_t(cur ^ 1) * cap;
#ifdef PF_CLUSTER_TRACE  // dev: per-warp phase clocks of one step (tools/cluster_trace.py)
        long long tr[5];
        tr[0] = clock64();
#endif
        // ---- S1: the slice's agents (listed at the previous step's start or
        // arrived since; those that left are empty now): proposals and claims.
        const uint32_t na = nagents[cur];
        for (uint32_t base = 0; base < na; base += NT) {
            const uint32_t e = base + threadIdx.x;
            const uint16_t ent = e < na ? agents_in[e] : uint16_t(0);
            const int r = entry_row(ent), lc = entry_col(ent);
            const uint32_t w = e < na ? word[at(r, lc)] : 0u;
            append(agents_out, &nagents[cur ^ 1], w != 0u, ent, cap, a.err);  // the next step's list
            int ic = -1;
            if (w != 0u) {
                const bool bottom = (w >> 30) == 2u;
                // Forward priority: no draw (src/lem.cpp:23-26).
                ic = slot_code(0, bottom);
                if (word[at(r + dr_of(ic), lc + dc_of(ic))] != 0u) {
                    uint32_t open = 0;
#pragma unroll
                    for (int i = 1; i < 8; ++i) {
                        const int c = slot_code(i, bottom);
                        open |= uint32_t(word[at(r + dr_of(c), lc + dc_of(c))] == 0u) << i;
                    }
                    ic = open == 0u ? -1 : slot_code(lem_choose_with(tab, open, seed, step, w & kIdMask), bottom);
                }
            }
            // Claim: OR the bit into the destination's byte; the first
            // claimer of a cell lists it with the cell's owner.
            bool first_local = false;
            uint16_t dest = 0;
            if (ic >= 0) {
                const int rd = r + dr_of(ic), ld = lc + dc_of(ic);
                const uint32_t bitv = 1u << (7 - ic);
                if (ld < 0) {
                    const int sh = 8 * ((cpc - 1) & 3);
                    if (((atomicOr(&claim_l[(rd * CP + cpc - 1) >> 2], bitv << sh) >> sh) & 0xFFu) == 0u) {
                        const uint32_t i = atomicAdd(&nclaims_l[cur], 1u);
                        if (i < uint32_t(cap)) claimed_l[i] = entry(rd, cpc - 1);
                        else atomicOr(a.err, 4u);
                    }
                } else if (ld >= ncols) {
                    if ((atomicOr(&claim_r[(rd * CP) >> 2], bitv) & 0xFFu) == 0u) {
                        const uint32_t i = atomicAdd(&nclaims_r[cur], 1u);
                        if (i < uint32_t(cap)) claimed_r[i] = entry(rd, 0);
                        else atomicOr(a.err, 4u);
                    }
                } else {
                    const int sh = 8 * (ld & 3);
                    first_local = ((atomicOr(&claim32[(rd * CP + ld) >> 2], bitv << sh) >> sh) & 0xFFu) == 0u;
                    dest = entry(rd, ld);
                }
            }
            append(claimed, &nclaims[cur], first_local, dest, cap, a.err);
        }
#ifdef PF_CLUSTER_TRACE
        tr[1] = clock64();
#endif
        cluster.sync();
#ifdef PF_CLUSTER_TRACE
        tr[2] = clock64();
#endif
        // ---- S2: resolution and commit at the claimed cells
        if (threadIdx.x == 0) {  // the lists of the next step: no reader or writer until the barrier
            nagents[cur] = 0u;
            nclaims[cur ^ 1] = 0u;
        }
        const uint32_t nc = nclaims[cur];
        for (uint32_t base = 0; base < nc; base += NT) {
            const uint32_t e = base + threadIdx.x;
            bool arrived = false;
            uint16_t ent = 0;
            if (e < nc) {
                ent = claimed[e];
                const int r = entry_row(ent), lc = entry_col(ent);
                const uint32_t cl8 = claim8[r * CP + lc];
                claim8[r * CP + lc] = 0u;
                const int grow = a.row_begin + r;
                const uint64_t gidx = uint64_t(grow) * uint64_t(W) + uint64_t(c_lo + lc);
                const int j = resolve(cl8, seed, step, gidx);
                const int rs = r + dr_of(j), ls = lc + dc_of(j);
                const uint32_t sw = word[at(rs, ls)];
                // Clear the source, its owner's copy and the ghost copies.
                word[at(rs, ls)] = 0u;
                if (ls < 0) {
                    word_l[at(rs, cpc - 1)] = 0u;
                } else if (ls >= ncols) {
                    word_r[at(rs, 0)] = 0u;
                } else {
                    if (ls == 0 && word_l) word_l[at(rs, cpc)] = 0u;
                    if (ls == ncols - 1 && word_r) word_r[at(rs, -1)] = 0u;
                }
                const uint32_t group = sw >> 30;
                uint32_t nw = sw;
                if (!(sw & kCrossedBit) && crossed_at(group, grow, a.k.H, band)) {  // src/engine.cpp:163-170
                    nw |= kCrossedBit;
                    if (group == 1u) ++ntop;
                    else ++nbot;
                }
                ++moved;
                word[at(r, lc)] = nw;
                if (lc == 0 && word_l) word_l[at(r, cpc)] = nw;
                if (lc == ncols - 1 && word_r) word_r[at(r, -1)] = nw;
                arrived = true;
            }
            append(agents_out, &nagents[cur ^ 1], arrived, ent, cap, a.err);
        }
        moved = __reduce_add_sync(0xFFFFFFFFu, moved);
        ntop = __reduce_add_sync(0xFFFFFFFFu, ntop);
        nbot = __reduce_add_sync(0xFFFFFFFFu, nbot);
        if (lane == 0 && (moved | ntop | nbot)) {
            atomicAdd(&cnt[s][0], moved);
            atomicAdd(&cnt[s][1], ntop);
            atomicAdd(&cnt[s][2], nbot);
        }
        moved = ntop = nbot = 0u;
#ifdef PF_CLUSTER_TRACE
        tr[3] = clock64();
#endif
        cluster.sync();
#ifdef PF_CLUSTER_TRACE
        tr[4] = clock64();
        if (s == n / 2 && (q == 0 || q == 7) && lane == 0)
            printf("TRACE step %u cta %d warp %d na %u nc %u  S1 %lld  bar1 %lld  S2 %lld  bar2 %lld\n", step, q, warp,
                   nagents[cur ^ 1], nc, tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3]);
#endif
    }
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");
    // The launch's counters go to the report ring (no global memory traffic
    // inside the step loop: a cluster barrier's release would wait for it).
    for (int t = threadIdx.x; t < n; t += NT) {
        const uint32_t step = step0 + uint32_t(t);
        uint32_t* const slot = a.reports + (size_t(rep) * a.report_cap + step % uint32_t(a.report_cap)) * 4;
        if (q == 0) slot[0] = step;
        if (cnt[t][0]) atomicAdd(&slot[1], cnt[t][0]);
        if (cnt[t][1]) atomicAdd(&slot[2], cnt[t][1]);
        if (cnt[t][2]) atomicAdd(&slot[3], cnt[t][2]);
    }
    // Write back the words (0 where empty) and the occupancy planes of the
    // final parity, 32-column segments spread over the cluster's CTAs (a
    // segment's words may live in two slices: read through DSMEM); bits of
    // columns >= W (the last segment's padding) are kept.
    uint2* const occ_out = a.p.occ[parity ^ (n & 1)] + size_t(rep) * a.p.occ_plane;
    const int segs = (W + 31) / 32;
    for (int sg = q; sg < segs; sg += cl) {
        const int c = 32 * sg + lane;
        const int owner = min(c, W - 1) / cpc;
        const uint32_t* const src = owner == q ? word : cluster.map_shared_rank(word, owner);
        for (int r = warp; r < H; r += NW) {
            const size_t b = size_t(kGhost + r);
            const uint32_t w = c < W ? src[at(r, c - owner * cpc)] : 0u;
            if (c < W) cw[b * W + c] = w;
            const uint32_t v30 = __ballot_sync(0xFFFFFFFFu, (w >> 30) & 1u);
            const uint32_t v31 = __ballot_sync(0xFFFFFFFFu, (w >> 31) & 1u);
            if (lane == 0) {
                const uint32_t valid = W - 32 * sg >= 32 ? 0xFFFFFFFFu : (1u << (W - 32 * sg)) - 1u;
                const uint2 p = occ_in[b * wsp + sg + 2];
                occ_out[b * wsp + sg + 2] = make_uint2((p.x & ~valid) | (v30 & valid), (p.y & ~valid) | (v31 & valid));
            }
        }
    }
    cluster.sync();  // no CTA leaves while another still reads its words
}

// The cluster size for this context, or 0 when the path does not apply:
// LEM, an unsharded grid, every replica a cluster resident at once (the
// replica batches keep the bit-plane kernel, which fills the GPU).
static Geometry geometry(const StepArgs& a, int cl, uint32_t max_agents) {
    const int cpc = (a.k.W + cl - 1) / cl;
    // A list holds distinct cells of the slice: the step-start agents (some of
    // which leave) plus the arrivals, so at most twice the agents.
    const int cap = int(std::min<long long>(2LL * max_agents, (long long)a.rows_owned * cpc));
    int cb = 1;
    while ((1 << cb) < cpc) ++cb;
    return Geometry{cl, cpc, cb, cap, smem_bytes(a.rows_owned, cpc, cap)};
}

}  // namespace cluster_lem

// The kernel instantiation for a thread count.
static auto kernel_for(int nt) { return nt == 512 ? cluster_lem::lem_cluster_kernel<512> : cluster_lem::lem_cluster_kernel<1024>; }

int plan_cluster_lem(const StepArgs& a, uint32_t max_agents, int* cap, int* nt) {
    using namespace cluster_lem;
    if (a.k.model != 0 || a.small_tiles == 1) return 0;
    if (a.row_begin != 0 || a.rows_owned != a.k.H) return 0;
    const char* env = std::getenv("PEDFLOW_CLUSTER");  // dev: 0 = off
    if (env && std::atoi(env) == 0) return 0;
    // 16 SMs issue the proposals: dense grids keep the whole GPU (bit-plane
    // kernel). Cut from tools/cluster_sweep.py.
    const char* dens = std::getenv("PEDFLOW_CLUSTER_MAX_DENSITY");  // dev override
    const double max_density = dens ? std::atof(dens) : kMaxDensity;
    if (double(max_agents) > max_density * double(a.k.W) * double(a.k.H)) return 0;
    for (int t : {512, 1024})
        if (cudaFuncSetAttribute(kernel_for(t), cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
    // Replicas beyond the resident clusters run in waves (one replica per
    // cluster for the whole launch): take the cluster size with the fewest
    // waves, 16 CTAs on a tie.
    int best = 0;
    long long best_waves = 0;
    const char* csz = std::getenv("PEDFLOW_CLUSTER_SIZE");  // dev: 16 or 8 only
    for (int cl : {16, 8}) {
        if (csz && std::atoi(csz) != cl) continue;
        const Geometry g = geometry(a, cl, max_agents);
        // Slices of at least 2 columns: a remote source clear then has exactly
        // one ghost copy (the clearing CTA's own).
        if (g.bytes > kSmemMax || g.cpc < 2 || a.rows_owned >= (1 << (16 - g.cb))) continue;
        const int threads = max_agents <= 512u * uint32_t(cl) ? 512 : 1024;
        const auto kernel = kernel_for(threads);
        if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(g.bytes)) !=
            cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(cl * a.replicas));
        cfg.blockDim = dim3(unsigned(threads));
        cfg.dynamicSmemBytes = g.bytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(cl);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kernel, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (clusters < 1) continue;
        const long long waves = (a.replicas + clusters - 1) / clusters;
        if (best == 0 || waves < best_waves) {
            best = cl;
            best_waves = waves;
            *cap = g.cap;
            *nt = threads;
        }
    }
    const double batch_density = dens ? max_density : kMaxDensityBatch;
    if (a.replicas > 1 &&
        (best_waves > kMaxWaves || double(max_agents) > batch_density * double(a.k.W) * double(a.k.H)))
        return 0;
    return best;
}

// a.nsteps steps as one cluster-resident launch; returns the launches issued.
int launch_cluster_lem(const StepArgs& a, int slot_idx, int parity, cudaStream_t s) {
    using namespace cluster_lem;
    if (a.nsteps > kMaxSteps || a.nsteps < kMinSteps) return 0;
    Geometry g = geometry(a, a.cluster, 0);
    g.cap = a.cluster_cap;
    g.bytes = smem_bytes(a.rows_owned, g.cpc, g.cap);
    // (replicas beyond the resident clusters queue: waves)
    // The attribute is per function; another context may have planned a
    // smaller footprint since.
    const auto kernel = kernel_for(a.cluster_nt);
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(g.bytes)) != cudaSuccess)
        return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(g.cl * a.replicas));
    cfg.blockDim = dim3(unsigned(a.cluster_nt));
    cfg.dynamicSmemBytes = g.bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(g.cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, kernel, a, slot_idx, parity, g.cpc, g.cap, g.cb) != cudaSuccess) {
        cudaGetLastError();
        return 0;  // the bit-plane kernel takes the step
    }
    return 1;
}

}  // namespace pfk
