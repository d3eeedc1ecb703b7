// Bit-sliced fused step kernel on occupancy bit planes (the default product
// path, PF_KERNEL_FUSED).
//
// State representation:
//   occ[parity]  ping-pong occupancy bit planes, one uint2 {v30, v31} per
//                32-cell row segment: bit j of v30 / v31 is bit 30 / 31 of the
//                cell word of column 32*seg + j (Top = v30 & ~v31, Bottom =
//                v31 & ~v30, Empty = ~(v30 | v31), wall = both). Rows are
//                padded with two wall segments on each side, so a strip's
//                plane window is one aligned run of NS + 4 segments.
//   cell         the 32-bit cell words (id | crossed | group), updated IN
//                PLACE and meaningful only where the planes say "occupied":
//                a step reads words only at cells occupied at its start
//                (draw keys, arrival sources) and writes them only at cells
//                empty at its start (arrivals), so the two sets never meet
//                and no ping-pong copy of the 4 B/cell words is needed.
//                Vacated cells keep a stale word; state export masks words
//                with the planes (launch_sanitize_words).
//
// The per-step update (StepEngine::step, src/engine.cpp:53-193) is evaluated
// on 32-cell row segments held as 32-bit masks, so the common work costs one
// ALU op per 32 cells; only agents that must draw (forward blocked, some slot
// open) and destinations with >= 2 claimants fall to per-cell scalar code, and
// those are compacted into shared-memory work lists so every lane takes one.
//
// Persistent column sweep: a CTA owns a strip of NS 32-column segments and a
// run of consecutive RT-row tiles. The step-start planes of the strip live in
// a shared-memory ring of staged rows (tile + 3-row halo + the next tile's
// rows); while a tile is processed, TMA bulk copies (cp.async.bulk + mbarrier,
// one (NS + 4) * 8-byte row each) bring the next tile's RT new rows. One warp
// claims work items from a per-step counter and publishes them decoded.
//
//   S1 intent  thread per segment-row: forward moves (F open, no draw,
//              src/lem.cpp:23-26, src/aco.cpp:60-63) and boxed-in agents in
//              bit logic; agents that must draw are queued, then run the
//              scalar LEM / ACO selection one per thread with the open-slot
//              mask built from the planes. Output: 8 intent planes D_j (bit
//              set: the agent there moves toward row-major direction j).
//   S2 resolve thread per segment-row: claims C_k on every destination from
//              the shifted intent planes (the gather of src/engine.cpp:101-122,
//              row-major contender order), at-least-two detection in bit logic;
//              contested cells are queued for the keyed draw. Winner code
//              planes (A, K0..K2); granted moves are OR-ed onto the sources.
//   S3 commit  warp per row, lane = column: arrivals (source word, crossing,
//              counters, tour), the new occupancy planes (vacates cleared,
//              arrivals set by group ballots), ACO evaporation + deposit over
//              every cell (src/engine.cpp:124-175).
//
// Linked row shards (MIRROR): boundary items are claimed first, wait for the
// neighbour's previous-step boundary items, copy their edge rows into the
// neighbour's ghost rows (peer memory) and count themselves toward the flag
// that releases the neighbour's next step (wait_boundary / mirror_tile /
// signal_boundary below).
//
// This file is the kernel template: it is compiled once per strip width
// (pf_bitstep_ns8.cu: 8 segments = 256 columns, pf_bitstep_ns10.cu: 320
// columns), each into its own namespace; pf_bitstep.cu picks one per grid
// width (bits_strip_segments).
#include <algorithm>
#include <cstddef>

#include "pf_internal.h"

#ifndef PF_BITS_NAMESPACE
#error "define PF_BITS_NS and PF_BITS_NAMESPACE before including pf_bitstep.cuh"
#endif

namespace pfk {
namespace PF_BITS_NAMESPACE {

using namespace pfdev;

namespace {

#ifndef PF_BITS_RT
#define PF_BITS_RT 16
#endif
#ifndef PF_BITS_NS
#define PF_BITS_NS 8
#endif
#ifndef PF_BITS_NT
#define PF_BITS_NT 256
#endif
constexpr int RT = PF_BITS_RT;   // output rows per tile
constexpr int NS = PF_BITS_NS;   // output 32-column segments per strip
constexpr int SR = RT + 6;       // staged rows of one tile: -3 .. RT+2
#ifdef PF_BITS_SMALL_RING  // debug build (tools/build_debug.sh): no cross-item prefetch
#define PF_BITS_RING (SR + RT)
#endif
#ifndef PF_BITS_RING
#define PF_BITS_RING (2 * SR)
#endif
// Ring slots: the current window + the next tile's rows, or (2 * SR) the next
// item's whole window, prefetched during an item's last tile.
constexpr int RING = PF_BITS_RING;
constexpr bool kCrossPrefetch = RING >= 2 * SR;
static_assert(RING >= SR + RT, "the ring must hold a window and the next tile's rows");
constexpr int SS = NS + 2;       // intent / resolution segments: -1 .. NS
constexpr int SP = NS + 4;       // staged plane segments: -2 .. NS+1 (pl index = si + 1)
static_assert(SP * 8 % 16 == 0, "a staged plane row must be a whole number of 16-byte TMA units");
constexpr int NT = PF_BITS_NT;   // threads per CTA
// Resident CTAs per SM (register budget 65536 / (NT * CTAS)), chosen per
// launch (see launch()): 4 (64 registers) for LEM and for small
// replica-batched ACO grids; 3 (80 registers, no spills) for large ACO grids,
// which are pure pheromone streams; 5 (48 registers) for large LEM grids.
constexpr int kRegCtas = NT == 256 ? 4 : 65536 / (NT * 64);
constexpr int NW = NT / 32;
constexpr int DROWS = RT + 4;    // intent rows -2 .. RT+1
constexpr int AROWS = RT + 2;    // resolution rows -1 .. RT
constexpr int NU = DROWS * SS;   // intent units (>= resolution units AROWS * SS)
// The warp that issues the row loads and claims work items during the tile
// loop: the last one. S1 units fill the warps in order, so the last warp has
// the fewest (or none) and its issue work does not delay the S1 barrier.
constexpr int kIoWarp = NW - 1;
static_assert(NU * 32 < (1 << 16), "work-list bit counts must fit 16 bits");

struct Smem {
    uint2 pl[RING][SP];             // staged {v30, v31} planes; pl[.][si + 1] = segment si
    uint32_t D[8][DROWS][SS + 2];   // intent planes, D[.][.][si + 1]; the end columns stay 0
    uint32_t A[AROWS][SS];
    uint32_t K[3][AROWS][SS];
    uint32_t G[2][RT][SS];          // grants (vacates) onto owned rows, double-buffered per tile
    uint32_t rowdraw[2][DROWS];     // intent row has a drawing agent (non-forward intents), per tile parity
    uint32_t dirty[2][RT];          // owned row has an arrival or a vacate
    // Scalar work list (S1 draws, then reused for S2 contested cells): one
    // entry per unit with work, in the order a packed counter handed out
    // (entry count << 16 | bit count, one native 32-bit shared atomic; at
    // most NU * 32 < 2^16 bits), so qp (first rank of the entry) is sorted
    // and rank r maps to its (unit, bit) by binary search. Bounded by the
    // unit count: it cannot overflow.
    uint32_t qu[NU];  // unit
    uint32_t qm[NU];  // its bits
    uint32_t qp[NU];  // rank of its first bit
    // S3: per warp, the words (and ACO tours, then deposits) at the sources
    // of its row's arrivals, by arrival, fetched at once by cp.async.
    uint32_t asw[NW][NS][32];
    uint16_t alist[NW][NS * 32];  // S3: the row's arrivals (column | direction code << 12), per warp
    unsigned long long mbar[2];
    uint32_t qc[2][2];  // [tile parity][0: S1 draws, 1: S2 contested cells]
    // Next work item. Double-buffered by the parity of the item that claims it:
    // with one-tile items the next claim can come before the slowest warp
    // has read the previous one (no barrier in between).
    int item[2];
    int idec[2][5];   // the same items decoded (rep, strip, chunk, sides, step offset) once: no divisions per thread
    int defer[2];     // multi-step launches: the item's window could not be prefetched (dependencies pending)
    uint32_t cnt[3];
    double atr[NW][NS][32];  // ACO only: LEM launches allocate the struct without it (last member)
};
constexpr size_t kSmemBytes[2] = {offsetof(Smem, atr), sizeof(Smem)};  // [ACO]

__device__ __forceinline__ uint32_t bit(uint32_t x, int j) { return (x >> j) & 1u; }

// Value of a plane at column c-1 (shift in from the left segment) / c+1.
__device__ __forceinline__ uint32_t from_left(uint32_t x, uint32_t left) { return (x << 1) | (left >> 31); }
__device__ __forceinline__ uint32_t from_right(uint32_t x, uint32_t right) { return (x >> 1) | (right << 31); }

// --- TMA bulk copy (cp.async.bulk) + mbarrier ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(m))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, uint32_t parity) {
    asm volatile(
        "{\n"
        "  .reg .pred done;\n"
        "WAIT_%=:\n"
        "  mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "  @!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}

// --- cp.async (LDGSTS) of single words into shared memory ----------------
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Ring slot of staged row sr (0 = tile row -3) for a window starting at base.
__device__ __forceinline__ int slot(int base, int sr) {
    const int s = base + sr;
    return s >= RING ? s - RING : s;
}

__device__ __forceinline__ uint32_t empty_of(uint2 p) { return ~(p.x | p.y); }

// Pheromone storage per cell: {top, bottom} as fp64 (double2, the product,
// bit-exact) or fp32 (float2, PF_KERNEL_FUSED_F32, tolerance-only). All
// arithmetic is fp64 (the reference's order and rounding); an fp32 store
// rounds the result once.
template <class TV> struct Tau;
template <> struct Tau<double2> {
    using S = double;
    __device__ __forceinline__ static double2 make(double a, double b) { return make_double2(a, b); }
};
template <> struct Tau<float2> {
    using S = float;
    __device__ __forceinline__ static float2 make(double a, double b) {
        return make_float2(__double2float_rn(a), __double2float_rn(b));
    }
};
template <class TV>
__device__ __forceinline__ TV evaporated(TV t, double f) {
    return Tau<TV>::make(__dmul_rn(double(t.x), f), __dmul_rn(double(t.y), f));
}

// Emptiness around one intent unit: the eight neighbour planes, shifted so
// bit j is the neighbour of column j.
struct Around {
    uint32_t em, emL, emR, e0L, e0R, ep, epL, epR;
};

__device__ __forceinline__ Around around(const Smem& sm, int base, int sr, int si) {
    const uint2* rm = sm.pl[slot(base, sr - 1)] + si + 1;
    const uint2* r0 = sm.pl[slot(base, sr)] + si + 1;
    const uint2* rp = sm.pl[slot(base, sr + 1)] + si + 1;
    Around n;
    n.em = empty_of(rm[0]);
    n.ep = empty_of(rp[0]);
    const uint32_t e0 = empty_of(r0[0]);
    n.emL = from_left(n.em, empty_of(rm[-1]));
    n.emR = from_right(n.em, empty_of(rm[1]));
    n.e0L = from_left(e0, empty_of(r0[-1]));
    n.e0R = from_right(e0, empty_of(r0[1]));
    n.epL = from_left(n.ep, empty_of(rp[-1]));
    n.epR = from_right(n.ep, empty_of(rp[1]));
    return n;
}

// Claims on the destinations of resolution unit (row ai-1, segment si).
__device__ __forceinline__ void claims(const Smem& sm, int ai, int si, uint32_t (&C)[8]) {
    const int dm = ai, d0 = ai + 1, dp = ai + 2;  // intent rows of rr-1, rr, rr+1
    auto D = [&](int k, int row, int s) -> uint32_t { return sm.D[k][row][s + 1]; };
    C[0] = from_left(D(7, dm, si), D(7, dm, si - 1));
    C[1] = D(6, dm, si);
    C[2] = from_right(D(5, dm, si), D(5, dm, si + 1));
    C[3] = from_left(D(4, d0, si), D(4, d0, si - 1));
    C[4] = from_right(D(3, d0, si), D(3, d0, si + 1));
    C[5] = from_left(D(2, dp, si), D(2, dp, si - 1));
    C[6] = D(1, dp, si);
    C[7] = from_right(D(0, dp, si), D(0, dp, si + 1));
    const uint32_t segmask = si == 0 ? 0x80000000u : (si == SS - 1 ? 0x00000001u : 0xFFFFFFFFu);
#pragma unroll
    for (int k = 0; k < 8; ++k) C[k] &= segmask;
}

// OR the source-grant bits of winners `wk` (direction k) at destination row
// rr of segment si into G.
__device__ __forceinline__ void grant(Smem& sm, int cur, int rr, int si, int k, uint32_t wk) {
    const int g = rr + kDR[k];
    if (g < 0 || g >= RT) return;
    sm.dirty[cur][g] = 1u;
    const int dc = kDC[k];
    if (dc == 0) {
        atomicOr(&sm.G[cur][g][si], wk);
    } else if (dc < 0) {
        atomicOr(&sm.G[cur][g][si], wk >> 1);
        if ((wk & 1u) && si > 0) atomicOr(&sm.G[cur][g][si - 1], 0x80000000u);
    } else {
        atomicOr(&sm.G[cur][g][si], wk << 1);
        if ((wk >> 31) && si + 1 < SS) atomicOr(&sm.G[cur][g][si + 1], 1u);
    }
}

// Flat form of the work list: one u16 (unit << 5 | bit) per listed bit, by
// rank, in the per-warp S3 buffers (free during S1/S2; the end-of-tile
// barrier separates their uses). A list longer than kFlatCap (it cannot be
// at realistic densities, but no bound rules it out) falls back to the
// binary search over the entries.
// Throughput geometries only (C3 x64 -6%, C4 x64 -3.6%): in the latency-bound
// small-grid geometry the producer's per-bit loop lengthens the slowest S1
// thread (singles +8%), so it keeps the search.
constexpr bool kFlat = NS >= 8;
constexpr int kFlatCap = kFlat ? int((sizeof(uint32_t) * NW * NS * 32 + sizeof(uint16_t) * NW * NS * 32) / sizeof(uint16_t)) : 0;
static_assert(NU < (1 << 11), "unit index must fit the flat list's 11 bits");
__device__ __forceinline__ uint16_t* flat_list(Smem& sm) { return reinterpret_cast<uint16_t*>(&sm.asw[0][0][0]); }
__device__ __forceinline__ const uint16_t* flat_list(const Smem& sm) {
    return reinterpret_cast<const uint16_t*>(&sm.asw[0][0][0]);
}

// Add unit u's bits `mask` to work list `list` (FLAT: also per-bit entries).
template <bool FLAT>
__device__ __forceinline__ void enqueue(Smem& sm, uint32_t* qc, int u, uint32_t mask) {
    const uint32_t old = atomicAdd(qc, (1u << 16) | uint32_t(__popc(mask)));
    const int e = int(old >> 16);
    sm.qu[e] = uint32_t(u);
    sm.qm[e] = mask;
    sm.qp[e] = old & 0xFFFFu;
    uint16_t* fl = flat_list(sm);
    if (FLAT)
        for (int k = int(old & 0xFFFFu); mask && k < kFlatCap; ++k) {
            fl[k] = uint16_t(u << 5 | (__ffs(mask) - 1));
            mask &= mask - 1u;
        }
}

// Position of the k-th (0-based) set bit of m.
__device__ __forceinline__ int nth_bit(uint32_t m, int k) {
    int pos = 0;
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const int c = __popc(m & ((1u << w) - 1u));
        if (k >= c) {
            k -= c;
            m >>= w;
            pos += w;
        }
    }
    return pos;
}

// Work-list rank r -> (unit, bit), n entries, nq bits.
template <bool FLAT>
__device__ __forceinline__ void list_entry(const Smem& sm, uint32_t n, uint32_t nq, uint32_t r, int& u, int& j) {
    if (FLAT && nq <= uint32_t(kFlatCap)) {
        const uint32_t v = flat_list(sm)[r];
        u = int(v >> 5);
        j = int(v & 31u);
        return;
    }
    int lo = 0, hi = int(n) - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sm.qp[mid] <= r) lo = mid;
        else hi = mid - 1;
    }
    u = int(sm.qu[lo]);
    j = nth_bit(sm.qm[lo], int(r - sm.qp[lo]));
}

}  // namespace

// Intent of the draw-path agent at bit j of intent unit (di, si):
// lem_select / aco_select (src/lem.cpp:28-60, src/aco.cpp:64-92). The agent's
// id (the selection key, src/engine.cpp:82) is read from its cell word: the
// cell is occupied at step start, so no thread writes it during this step.
template <bool ACO, class TV>
__device__ __forceinline__ int draw_intent(const StepArgs& a, const Smem& sm, int base, const uint32_t* cells,
                                           const TV* __restrict__ tin, int di, int si, int j, bool bottom,
                                           int r0, int c0, uint64_t seed, uint32_t step) {
    const int sr = di + 1;
    const int W = a.k.W;
    const int b = kGhost + r0 + di - 2;
    const int c = c0 + 32 * (si - 1) + j;
    const uint32_t id = cells[size_t(b) * W + c] & kIdMask;
    const Around n = around(sm, base, sr, si);
    uint32_t open;  // goal-relative slots F FL FR L R B BL BR
    if (!bottom)
        open = bit(n.ep, j) | bit(n.epL, j) << 1 | bit(n.epR, j) << 2 | bit(n.e0L, j) << 3 | bit(n.e0R, j) << 4 |
               bit(n.em, j) << 5 | bit(n.emL, j) << 6 | bit(n.emR, j) << 7;
    else
        open = bit(n.em, j) | bit(n.emR, j) << 1 | bit(n.emL, j) << 2 | bit(n.e0R, j) << 3 | bit(n.e0L, j) << 4 |
               bit(n.ep, j) << 5 | bit(n.epR, j) << 6 | bit(n.epL, j) << 7;
    int s;
    if (!ACO) {
        s = lem_choose(a.kc, open, seed, step, id);
    } else {
        // All the open neighbours' loads are issued before any is used. Only
        // open slots are read: an open slot is an empty cell inside the
        // buffer, while a closed one may lie outside it (an agent in a
        // shard's first ghost row at column 0 has its (-1,-1) neighbour
        // before the start of the allocation).
        using S = typename Tau<TV>::S;
        const S* t0 = reinterpret_cast<const S*>(tin + size_t(b) * W + c) + (bottom ? 1 : 0);
        // Goal-relative slot offsets of a Top agent (inc/grid.hpp:19-43); a
        // Bottom agent's are their point reflection (inc/grid.hpp:45-49).
        constexpr int kSlotDR[8] = {1, 1, 1, 0, 0, -1, -1, -1};
        constexpr int kSlotDC[8] = {0, -1, 1, -1, 1, 0, -1, 1};
        // Interleaved {top, bottom}: a neighbour (dr, dc) is 2 * (dr * W + dc)
        // scalars away; the three rows' pointers and the column step are
        // formed once.
        const ptrdiff_t c2 = bottom ? -2 : 2, r2 = c2 * W;
        const S* rows[3] = {t0 - r2, t0, t0 + r2};  // goal-relative rows dr = -1, 0, +1
        double tn[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            tn[i] = (open >> i & 1u) ? double(__ldg(rows[kSlotDR[i] + 1] + c2 * kSlotDC[i])) : 0.0;
        // aco_numerators (src/aco.cpp:39-51), the alpha case taken once.
        double num[8];
        const int mode = __ldg(&a.kc->alpha_mode);
        if (mode == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) num[i] = (open >> i & 1u) ? __dmul_rn(tn[i], a.k.eta[i]) : 0.0;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                num[i] = (open >> i & 1u) ? __dmul_rn(pheromone_term(a.kc, tn[i]), a.k.eta[i]) : 0.0;
        }
        s = aco_choose(num, open, seed, step, id);
    }
    // Slot -> row-major code: kSlotCodeTop packed in nibbles (6,5,7,3,4,1,0,2),
    // a Bottom agent's code is 7 - that.
    const int code = int((0x20143756u >> (4 * s)) & 7u);
    return bottom ? 7 - code : code;
}

// Keyed draw for a contested destination at bit j of resolution unit (ai, si):
// the winner's row-major code (src/engine.cpp:116-120).
__device__ __forceinline__ int draw_winner(const StepArgs& a, const Smem& sm, int ai, int si, int j, int r0, int c0,
                                           uint64_t seed, uint32_t step) {
    uint32_t C[8];
    claims(sm, ai, si, C);
    uint32_t m = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) m |= bit(C[k], j) << k;
    const int64_t grow = int64_t(a.row_begin) + r0 + ai - 1;
    const int gcol = c0 + 32 * (si - 1) + j;
    return resolve(m, seed, step, uint64_t(grow) * uint64_t(a.k.W) + uint64_t(gcol));
}

__device__ __forceinline__ void set_winner(Smem& sm, int cur, int ai, int si, int j, int k) {
    const uint32_t b = 1u << j;
    if (k & 1) atomicOr(&sm.K[0][ai][si], b);
    if (k & 2) atomicOr(&sm.K[1][ai][si], b);
    if (k & 4) atomicOr(&sm.K[2][ai][si], b);
    grant(sm, cur, ai - 1, si, k, b);
}

// One work item: a chunk of consecutive RT-row tiles of one strip of one
// replica.
struct Item {
    int rep, strip, chunk, c0, t_first, t_end;
    int sl;     // step of the item relative to the launch's first step (multi-step launches)
    int sides;  // bit 0 / 1: the item reads the upper / lower ghost rows (and writes the rows they mirror)
};

// Ghost-row sides of a chunk: its first tile's window starts above row 0, or
// its last tile's window (RT rows + 3) reaches past the last owned row. With
// a short last tile that can be the last TWO chunks' business.
__device__ __forceinline__ int chunk_sides(int chunk, int tiles_per_item, int n_tiles, int rows_owned) {
    const int t0 = chunk * tiles_per_item, t1 = min(t0 + tiles_per_item, n_tiles);
    return (t0 == 0 ? 1 : 0) | (t1 * RT + kGhost > rows_owned ? 2 : 0);
}
// Items per replica-strip with side s (the count signal_boundary waits for).
__device__ __forceinline__ int side_chunks(int s, int n_chunks, int tiles_per_item, int n_tiles, int rows_owned) {
    int n = 0;
    for (int c = n_chunks - 1; c >= 0 && c >= n_chunks - 2; --c) n += chunk_sides(c, tiles_per_item, n_tiles, rows_owned) >> 1 & 1;
    return s == 0 ? 1 : n;
}

// Items are numbered strip-fastest, then replica, then chunk: the CTAs in
// flight at any moment work on a band of whole rows (of every replica of a
// batch) rather than on a few hundred tiles down one strip. For batches,
// replica before chunk takes the 480^2 x64 configs 9-16% faster than
// replica-major numbering.
// The stream then covers full rows of every plane: C5 ACO's DRAM bytes fall
// to the algorithmic 8.8 GB (neighbouring tiles' halo and draw reads hit in
// L2) and, mostly, the achieved DRAM bandwidth rises (the step runs 7.8%
// faster than with chunk-fastest numbering). Linked shards (bfirst) number the
// boundary chunks of every (replica, strip) first, so they are claimed early
// in the step: the neighbours' next steps wait only for those (see
// wait_boundary / signal_boundary).
// The k-th row band of chunks, taken alternately from the top and the bottom
// of the grid (0, n-1, 1, n-2, ...): the crowded bands at both ends start
// early and are spread over the step (C5 LEM -5.8%, C3 x64 -4.2%, ACO -1%).
// Used when there are more items than CTAs (decode_item's `spread`).
__device__ __forceinline__ int two_ended(int k, int n) { return (k & 1) ? n - 1 - (k >> 1) : (k >> 1); }

__device__ __forceinline__ Item decode_item(int item, int strips, int n_chunks, int n_tiles, int tiles_per_item,
                                            int reps, bool bfirst, int rows_owned, bool spread) {
    Item it;
    if (bfirst) {
        const int nb = n_chunks >= 2 ? 2 : 1, nbi = reps * strips * nb;
        if (item < nbi) {
            it.rep = item / (strips * nb);
            const int r = item % (strips * nb);
            it.strip = r / nb;
            it.chunk = (r % nb) ? n_chunks - 1 : 0;
        } else {
            const int j = item - nbi;
            it.strip = j % strips;
            it.rep = (j / strips) % reps;
            it.chunk = 1 + (spread ? two_ended(j / (strips * reps), n_chunks - nb) : j / (strips * reps));
        }
    } else {
        it.strip = item % strips;
        it.rep = (item / strips) % reps;
        it.chunk = spread ? two_ended(item / (strips * reps), n_chunks) : item / (strips * reps);
    }
    it.sides = bfirst ? chunk_sides(it.chunk, tiles_per_item, n_tiles, rows_owned) : 0;
    it.sl = 0;
    it.c0 = it.strip * (NS * 32);
    it.t_first = it.chunk * tiles_per_item;
    it.t_end = min(it.t_first + tiles_per_item, n_tiles);
    return it;
}

// An item decoded by the claiming warp (Smem::idec) for the rest of the CTA.
__device__ __forceinline__ void publish_item(int (&d)[5], const Item& it) {
    d[0] = it.rep;
    d[1] = it.strip;
    d[2] = it.chunk;
    d[3] = it.sides;
    d[4] = it.sl;
}
__device__ __forceinline__ Item read_item(const int (&d)[5], int n_tiles, int tiles_per_item) {
    Item it;
    it.rep = d[0];
    it.strip = d[1];
    it.chunk = d[2];
    it.sides = d[3];
    it.sl = d[4];
    it.c0 = it.strip * (NS * 32);
    it.t_first = it.chunk * tiles_per_item;
    it.t_end = min(it.t_first + tiles_per_item, n_tiles);
    return it;
}

// Multi-step launches (StepArgs::nsteps > 1, unlinked contexts): the launch
// runs nsteps consecutive steps and its CTAs claim items step-major from one
// counter, g = sl * n_items + i. An item of step step0 + sl > step0 starts
// once the 3x3 neighbourhood of its tiles (strips strip - 1 .. strip + 1,
// tiles t_first - 1 .. t_end; the step's dependency radius, 3 rows and 64
// columns, is within one tile and one strip) has completed the previous step:
// tile_done[rep][strip][tile] = last completed step + 1, released by the CTA
// that finished the tile. Steps thus overlap in the tail instead of
// draining the GPU at every step boundary. The reads and writes the wait
// orders are exactly those of the stream order between step launches:
// step s reads the neighbourhood's step s-1 output and overwrites the
// buffers (ping-pong planes, in-place words and tours at cells empty at step
// start) that the neighbourhood read during step s-1.
__device__ __forceinline__ Item decode_global(int g, int n_items, int strips, int n_chunks, int n_tiles,
                                              int tiles_per_item, int reps, bool bfirst, int rows_owned, bool spread,
                                              bool multi) {
    const int sl = multi ? g / n_items : 0;
    Item it = decode_item(g - sl * n_items, strips, n_chunks, n_tiles, tiles_per_item, reps, bfirst, rows_owned, spread);
    it.sl = sl;
    return it;
}

// Called by a full warp: are the neighbourhood's tiles done with step
// need - 1? With `block`, spins until they are (30 s timeout sets *a.err).
__device__ __forceinline__ bool deps_ready(const StepArgs& a, const Item& it, uint32_t need, int strips, int n_tiles,
                                           bool block) {
    const int lane = threadIdx.x & 31;
    const int s_lo = max(0, it.strip - 1), s_hi = min(strips - 1, it.strip + 1);
    const int t_lo = max(0, it.t_first - 1), t_hi = min(n_tiles - 1, it.t_end);
    const int nt = t_hi - t_lo + 1, total = (s_hi - s_lo + 1) * nt;
    uint64_t t0 = 0;
    for (;;) {
        bool ok = true;
        for (int k = lane; k < total; k += 32) {
            const uint32_t* f = a.tile_done + (size_t(it.rep) * strips + (s_lo + k / nt)) * n_tiles + (t_lo + k % nt);
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            ok = ok && int32_t(v - need) >= 0;
        }
        ok = __all_sync(0xFFFFFFFFu, ok);
        if (ok || !block) return ok;
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (!t0) t0 = now;
        uint32_t err;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(err) : "l"(a.err) : "memory");
        if (__any_sync(0xFFFFFFFFu, (err & 2u) != 0u)) return true;  // another wait timed out: drain
        if (now - t0 > 10000000000ull) {
            if (lane == 0) atomicOr(a.err, 2u);
            return true;
        }
        __nanosleep(64);
    }
}

// Issue the TMA loads of `nrows` staged plane rows (tile rows first_sr..,
// relative to the tile at r0) of item `it` into their ring slots, completing
// on mbarrier m; rows past the end of the buffer are written as walls. Each
// row is one 16-byte-aligned run of SP segments (the row padding holds walls
// beyond the grid's columns). Called by one full warp.
__device__ __forceinline__ void load_rows(Smem& sm, const StepArgs& a, int parity, const Item& it, int r0, int base,
                                          int first_sr, int nrows, unsigned long long* m) {
    const int lane = threadIdx.x & 31;
    const uint2* src = a.p.occ[parity] + size_t(it.rep) * a.p.occ_plane + size_t(it.strip) * NS;
    const int b_first = kGhost + r0 - 3 + first_sr;
    const int nvalid = max(0, min(nrows, a.rows_buf - b_first));
    if (lane == 0) mbar_expect_tx(m, uint32_t(nvalid) * uint32_t(SP * 8));
    __syncwarp();
    for (int i = lane; i < nvalid; i += 32)
        bulk_g2s(&sm.pl[slot(base, first_sr + i)][0], src + size_t(b_first + i) * a.p.wsp, uint32_t(SP * 8), m);
    for (int i = nvalid * SP + lane; i < nrows * SP; i += 32)
        sm.pl[slot(base, first_sr + i / SP)][i % SP] = make_uint2(kWall, kWall);
}

// Fused halo exchange, ordering (linked shards only). A boundary item of step
// t reads this shard's ghost rows (written by the neighbour's step t-1
// boundary items) and writes the neighbour's ghost rows of the other parity
// (read by the neighbour's step t-1 boundary items). Both hazards are covered
// by waiting, before the item's rows are loaded, until the neighbour has
// completed its step t-1 boundary items: sync_local[side] >= t. Interior
// items never wait, so neighbouring shards overlap everything but their
// boundary strips. Called by one lane; a 30 s timeout sets *err.
__device__ __forceinline__ void wait_boundary(const StepArgs& a, int sides, uint32_t step) {
    uint64_t t0 = 0;
    for (int s = 0; s < 2; ++s) {
        if (!(sides >> s & 1) || !a.peer[s].cell) continue;
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.sync_local + s) : "memory");
            if (int32_t(v - step) >= 0) break;
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (!t0) t0 = now;
            if (now - t0 > 30000000000ull) {  // the neighbour is gone
                atomicOr(a.err, 1u);
                return;
            }
            __nanosleep(200);
        }
    }
}

// After a boundary item (its mirror stores fenced, then a CTA barrier):
// count it; the CTA completing the last boundary item of a side releases
// step + 1 into that neighbour's flag. Called by one thread.
__device__ __forceinline__ void signal_boundary(const StepArgs& a, int sides, uint32_t step, int strips, int n_chunks,
                                                int n_tiles) {
    for (int s = 0; s < 2; ++s) {
        if (!(sides >> s & 1) || !a.peer[s].cell) continue;
        const uint32_t done = atomicAdd(a.bcount + size_t(step % uint32_t(a.report_cap)) * 2 + s, 1u) + 1u;
        if (done == uint32_t(strips * a.replicas * side_chunks(s, n_chunks, a.tiles_per_cta, n_tiles, a.rows_owned))) {
            __threadfence_system();
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.sync_remote[s]), "r"(step + 1u) : "memory");
        }
    }
}

// Fused halo exchange (linked shards only): after a tile's commit, its rows
// that are ghost rows of a neighbour shard (this shard's first / last kGhost
// owned rows) are copied from where the commit just wrote them (L2) into the
// neighbour's ghost rows: occupancy planes and pheromone of the new parity,
// words and tours in place (a stale word under an empty plane bit is as
// harmless there as here). Called by the whole CTA after the end-of-tile
// barrier; the system fence orders the stores before the step's completion
// flag (signal_boundary).
template <bool ACO, class TV>
__device__ __forceinline__ void mirror_tile(const StepArgs& a, int parity, int rep, int strip, int r0) {
    const int W = a.k.W;
    const int c0 = strip * NS * 32, ncols = min(NS * 32, W - c0);
    const size_t pb = size_t(rep) * a.p.plane, ob = size_t(rep) * a.p.occ_plane;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const PeerRows pr = a.peer[s];
        if (!pr.cell) continue;
        const int lo = max(r0, s == 0 ? 0 : a.rows_owned - kGhost);
        const int hi = min(min(r0 + RT, a.rows_owned), s == 0 ? kGhost : a.rows_owned);
        for (int lr = lo; lr < hi; ++lr) {
            const int b = kGhost + lr, pbr = b + pr.row_delta;
            const size_t src = pb + size_t(b) * W + c0, dst = size_t(rep) * pr.plane + size_t(pbr) * W + c0;
            for (int i = threadIdx.x; i < ncols; i += NT) {
                pr.cell[dst + i] = a.p.cell[0][src + i];
                if (ACO) {
                    pr.tour[dst + i] = a.p.tour[src + i];
                    reinterpret_cast<TV*>(pr.tau[parity ^ 1])[dst + i] = reinterpret_cast<const TV*>(a.p.tau[parity ^ 1])[src + i];
                }
            }
            if (threadIdx.x < NS) {
                const size_t q = size_t(strip) * NS + 2 + threadIdx.x;
                pr.occ[parity ^ 1][size_t(rep) * pr.occ_plane + size_t(pbr) * a.p.wsp + q] =
                    a.p.occ[parity ^ 1][ob + size_t(b) * a.p.wsp + q];
            }
        }
    }
    __threadfence_system();
}

// COMPACT: S3 per-arrival work on compacted arrival lists (dense, batched
// 480^2 grids: C4 x64 -6.4%); off for large grids, where arrivals are sparse
// and the per-segment form is 1-2% faster.
// MULTI: compiled with the multi-step (tile-dependency) logic; instantiated
// only for the dense-grid variants that launch() runs that way.
template <bool ACO, int CTAS, bool MIRROR, bool COMPACT, bool MULTI, class TV = double2>
__global__ void __launch_bounds__(NT, CTAS) step_bits_kernel(const StepArgs a, int slot_idx, int parity) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    const int W = a.k.W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int strips = (W + NS * 32 - 1) / (NS * 32);
    const int n_tiles = (a.rows_owned + RT - 1) / RT;
    const int n_chunks = (n_tiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
    const int n_items = strips * n_chunks * a.replicas;  // per step
    // Two-ended row bands only pay when items queue up; when every item has
    // its own CTA (small grids), plain order keeps neighbouring tiles on
    // neighbouring CTAs.
    const bool spread = n_items > int(gridDim.x);
    const bool multi = MULTI && !MIRROR && a.nsteps > 1;  // tile-level dependencies between the launch's steps
    // Flat draw queues (kFlat) except for large ACO grids, where the
    // pheromone stream bounds the step and the producer loop cost 0.7% at C5.
    constexpr bool FLAT = kFlat && (COMPACT || !ACO);
    const int n_all = n_items * (multi ? a.nsteps : 1);

    if (threadIdx.x == 0) {
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        fence_mbar_init();
        sm.cnt[0] = sm.cnt[1] = sm.cnt[2] = 0u;
        sm.qc[0][0] = sm.qc[0][1] = sm.qc[1][0] = sm.qc[1][1] = 0u;
    }
    for (int i = threadIdx.x; i < 2 * RT * SS; i += NT) (&sm.G[0][0][0])[i] = 0u;
    for (int i = threadIdx.x; i < 2 * DROWS; i += NT) (&sm.rowdraw[0][0])[i] = 0u;
    for (int i = threadIdx.x; i < 2 * RT; i += NT) (&sm.dirty[0][0])[i] = 0u;
    for (int i = threadIdx.x; i < 8 * DROWS; i += NT) {  // the zero end columns of the intent planes
        sm.D[i / DROWS][i % DROWS][0] = 0u;
        sm.D[i / DROWS][i % DROWS][SS + 1] = 0u;
    }
    // Work item = (replica, strip, chunk of tiles_per_cta consecutive tiles),
    // taken from a per-launch counter so heavy (crowded) chunks balance out.
    // The next item is claimed during the current item's last tile and its
    // first window is loaded into the other half of the ring meanwhile.
    // The counter of batch slot slot_idx is zeroed before the batch and no
    // other launch touches it, so the first claim needs no ordering.
    uint32_t* const work = a.work + slot_idx;
    // At most one item per CTA (single small grids): CTA b takes item b and
    // nothing is claimed (no counter round trips on the step's critical path).
    const bool one_each = n_all <= int(gridDim.x);
    int item = 0;
    if (one_each) {
        item = int(blockIdx.x);
    } else if (warp == 0) {
        if (lane == 0) item = int(atomicAdd(work, 1u));
        item = __shfl_sync(0xFFFFFFFFu, item, 0);
    }
    // Launched with programmatic stream serialization: everything above only
    // touches shared memory and this launch's own counter, so it overlaps the
    // previous step's tail; from here on the previous step's results (planes,
    // words, step counter) are complete and visible.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t step0 = *a.d_step + uint32_t(slot_idx);
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) sm.item[1] = item;
        if (item < n_all) {
            const Item first = decode_global(item, n_items, strips, n_chunks, n_tiles, a.tiles_per_cta, a.replicas, MIRROR, a.rows_owned, spread, multi);
            if (lane == 0) publish_item(sm.idec[1], first);
            if (MIRROR && first.sides && lane == 0) wait_boundary(a, first.sides, step0);
            if (multi && first.sl > 0) deps_ready(a, first, step0 + uint32_t(first.sl), strips, n_tiles, true);
            __syncwarp();
            load_rows(sm, a, parity ^ (first.sl & 1), first, first.t_first * RT, 0, 0, SR, &sm.mbar[0]);
        }
    }
    __syncthreads();  // item id and wall rows written by warp 0 are visible to all
    item = sm.item[1];
    int islot = 1;    // sm.idec slot of the current item
    int ipar = 0;     // the current item's last tile claims the next one into sm.item[ipar]
    uint32_t moved = 0, ntop = 0, nbot = 0;
    uint32_t nload = item < n_all ? 1u : 0u;    // load i completes mbar[i & 1], phase i >> 1
    int base = 0;                               // ring slot of staged row 0 of the current tile
    int cur = 0;                                // tile parity: G / dirty / work-list counters
    uint32_t* const cells = a.p.cell[0];
    while (item < n_all) {
    const Item it = read_item(sm.idec[islot], n_tiles, a.tiles_per_cta);
    const int rep = it.rep, c0 = it.c0;
    const uint32_t step = step0 + uint32_t(it.sl);  // this item's step and read parity
    const int par = parity ^ (it.sl & 1);
    const uint64_t seed = __ldg(&a.rep[rep].seed);
    const int band = __ldg(&a.rep[rep].band);
    const size_t plane_base = size_t(rep) * a.p.plane;
    uint32_t* const cw = cells + plane_base;
    uint2* const oout = a.p.occ[par ^ 1] + size_t(rep) * a.p.occ_plane + size_t(it.strip) * NS + 2;
    const TV* __restrict__ tin = ACO ? reinterpret_cast<const TV*>(a.p.tau[par]) + plane_base : nullptr;
    TV* __restrict__ tout = ACO ? reinterpret_cast<TV*>(a.p.tau[par ^ 1]) + plane_base : nullptr;
    double* __restrict__ tour = ACO ? a.p.tour + plane_base : nullptr;
    int next_base = 0;

    for (int t = it.t_first; t < it.t_end; ++t) {
        const int r0 = t * RT;               // owned-local row of the tile
        const uint32_t my_load = nload - 1;  // the load that brought this tile's new rows
        // Prefetch into the half of the ring this tile does not use (its
        // previous readers all passed the end-of-tile barrier): the next
        // tile's RT new rows, or on the last tile the next item's window.
        if (t + 1 < it.t_end) {
            if (warp == kIoWarp) load_rows(sm, a, par, it, r0 + RT, slot(base, RT), 6, RT, &sm.mbar[nload & 1]);
            ++nload;
        } else {
            next_base = kCrossPrefetch ? slot(base, SR) : 0;
            if (warp == kIoWarp) {
                int nx = 0;
                if (lane == 0) nx = one_each ? n_all : int(atomicAdd(work, 1u));
                nx = __shfl_sync(0xFFFFFFFFu, nx, 0);
                if (lane == 0) sm.item[ipar] = nx;
                // This CTA's last item: the next step's grid may be scheduled
                // (its CTAs wait in griddepcontrol.wait until this grid ends).
                if (nx >= n_all && lane == 0) asm volatile("griddepcontrol.launch_dependents;");
                if (nx < n_all) {
                    const Item nit = decode_global(nx, n_items, strips, n_chunks, n_tiles, a.tiles_per_cta, a.replicas, MIRROR, a.rows_owned, spread, multi);
                    if (lane == 0) publish_item(sm.idec[ipar], nit);
                    // Multi-step: prefetch only if the next item's neighbourhood
                    // is already done (it may include this very item, which
                    // finishes only after this tile); else load it after the
                    // item (a blocking wait is safe there).
                    const bool ready = !multi || nit.sl == 0 ||
                                       deps_ready(a, nit, step0 + uint32_t(nit.sl), strips, n_tiles, false);
                    if (lane == 0) sm.defer[ipar] = ready ? 0 : 1;
                    if (kCrossPrefetch && ready) {
                        if (MIRROR && nit.sides && lane == 0) wait_boundary(a, nit.sides, step0);
                        __syncwarp();
                        load_rows(sm, a, parity ^ (nit.sl & 1), nit, nit.t_first * RT, next_base, 0, SR, &sm.mbar[nload & 1]);
                    }
                }
            }
        }
        // Scratch of the NEXT tile (its last readers passed the previous
        // end-of-tile barrier; its first writers come after this tile's).
        for (int i = threadIdx.x; i < RT * SS; i += NT) (&sm.G[cur ^ 1][0][0])[i] = 0u;
        if (threadIdx.x < DROWS) sm.rowdraw[cur ^ 1][threadIdx.x] = 0u;
        if (threadIdx.x < RT) sm.dirty[cur ^ 1][threadIdx.x] = 0u;
        if (threadIdx.x == 0) sm.qc[cur ^ 1][0] = sm.qc[cur ^ 1][1] = 0u;
        mbar_wait(&sm.mbar[my_load & 1], (my_load >> 1) & 1u);

#ifndef PF_BITS_STREAM_ONLY
        // A window without agents (no cell with exactly one occupancy bit in
        // staged rows -3 .. RT+2; walls have both) needs no S1/S2: nothing can
        // arrive in or leave the tile's rows, so S3 takes the no-movement path
        // for every row (planes copied, ACO pheromone evaporated). The work
        // scratch of this tile is already zero. (The crowd-free middle of the
        // C5 grid, most of it early in a run.)
        // LEM on the 256/320-column geometries, when the starting bands cover
        // under 30% of the rows (StepArgs::skip_empty: C5 LEM -14%, C1 x64
        // -10%; C3 x64, whose bands cover 45%, would pay for the check). For
        // ACO the pheromone stream bounds the step (+1.7% at C5), and in the
        // small-grid geometry the check made ptxas spill (C4 single +20%).
        // (The window is SR consecutive ring rows of SP segments, possibly
        // wrapping: read as 16-byte segment pairs, SP being even.)
        constexpr bool kSkipEmpty = !ACO && NS >= 8;
        static_assert(SP % 2 == 0, "staged rows are whole 16-byte units");
        const bool check = kSkipEmpty && a.skip_empty;
        bool any_agent = !check;
        if (check) {
            const uint4* ring = reinterpret_cast<const uint4*>(&sm.pl[0][0]);
            for (int t = threadIdx.x; t < SR * SP / 2; t += NT) {
                int i = base * (SP / 2) + t;
                if (i >= RING * (SP / 2)) i -= RING * (SP / 2);
                const uint4 q = ring[i];
                any_agent |= ((q.x ^ q.y) | (q.z ^ q.w)) != 0u;
            }
        }
        const bool has_agents = !check || __syncthreads_or(any_agent);
        if (has_agents) {
            // ------------------------------------------------------------ S1
            // Intents for rows -2 .. RT+1, all staged segments (halo segments
            // only at the two columns next to the strip). A thread takes two
            // vertically adjacent units: they share two of their four staged
            // rows (12 plane loads instead of 18).
            static_assert(DROWS % 2 == 0, "S1 pairs intent rows");
            for (int u2 = threadIdx.x; u2 < (DROWS / 2) * SS; u2 += NT) {
                const int dp = u2 / SS, si = u2 - dp * SS;
                const int di0 = 2 * dp;  // intent rows di0, di0 + 1 = staged rows di0 + 1, di0 + 2
                uint32_t E[4][3];        // emptiness of staged rows di0 .. di0 + 3 at segments si-1, si, si+1
                uint2 P[2];
    #pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint2* row = sm.pl[slot(base, di0 + r)] + si + 1;
                    const uint2 m = row[0];
                    E[r][0] = empty_of(row[-1]);
                    E[r][1] = empty_of(m);
                    E[r][2] = empty_of(row[1]);
                    if (r == 1) P[0] = m;
                    if (r == 2) P[1] = m;
                }
                const uint32_t segmask = si == 0 ? 0xC0000000u : (si == SS - 1 ? 0x00000003u : 0xFFFFFFFFu);
    #pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int di = di0 + k, u = di * SS + si;
                    Around n;
                    n.em = E[k][1];
                    n.emL = from_left(E[k][1], E[k][0]);
                    n.emR = from_right(E[k][1], E[k][2]);
                    n.e0L = from_left(E[k + 1][1], E[k + 1][0]);
                    n.e0R = from_right(E[k + 1][1], E[k + 1][2]);
                    n.ep = E[k + 2][1];
                    n.epL = from_left(E[k + 2][1], E[k + 2][0]);
                    n.epR = from_right(E[k + 2][1], E[k + 2][2]);
                    const uint2 p = P[k];
                    const uint32_t T = p.x & ~p.y & segmask, B = p.y & ~p.x & segmask;
                    uint32_t d[8];
    #pragma unroll
                    for (int q = 0; q < 8; ++q) d[q] = 0u;
                    d[6] = T & n.ep;  // Top forward: (+1, 0)
                    d[1] = B & n.em;  // Bottom forward: (-1, 0)
                    const uint32_t any8 = n.ep | n.epL | n.epR | n.e0L | n.e0R | n.em | n.emL | n.emR;
                    const uint32_t slow = ((T & ~n.ep) | (B & ~n.em)) & any8;
                    if (slow) {
                        enqueue<FLAT>(sm, &sm.qc[cur][0], u, slow);
                        sm.rowdraw[cur][di] = 1u;
                    }
    #pragma unroll
                    for (int q = 0; q < 8; ++q) sm.D[q][di][si + 1] = d[q];
                }
            }
            __syncthreads();
            // Draws, spread evenly over the CTA (the barrier is skipped,
            // uniformly, when there are none).
            if (const uint32_t nq = sm.qc[cur][0] & 0xFFFFu) {
                const uint32_t ne = sm.qc[cur][0] >> 16;
                for (uint32_t e = threadIdx.x; e < nq; e += NT) {
                    int u, j;
                    list_entry<FLAT>(sm, ne, nq, e, u, j);
                    const int di = u / SS, si = u - di * SS;
                    const bool bottom = bit(sm.pl[slot(base, di + 1)][si + 1].y, j) != 0u;
                    const int code = draw_intent<ACO, TV>(a, sm, base, cw, tin, di, si, j, bottom, r0, c0, seed, step);
                    atomicOr(&sm.D[code][di][si + 1], 1u << j);
                }
                __syncthreads();
            }

            // ------------------------------------------------------------ S2
            // Claims, winners and grants for destinations in rows -1 .. RT.
            for (int u = threadIdx.x; u < AROWS * SS; u += NT) {
                const int ai = u / SS, si = u - ai * SS;  // ai = rr + 1
                if (!(sm.rowdraw[cur][ai] | sm.rowdraw[cur][ai + 1] | sm.rowdraw[cur][ai + 2])) {
                    // No agent in the three intent rows around these destinations
                    // drew: the only claims are forward moves, from the row above
                    // (Top, code 1) and the row below (Bottom, code 6).
                    const uint32_t segmask = si == 0 ? 0x80000000u : (si == SS - 1 ? 0x00000001u : 0xFFFFFFFFu);
                    const uint32_t c1 = sm.D[6][ai][si + 1] & segmask, c6 = sm.D[1][ai + 2][si + 1] & segmask;
                    const uint32_t twos = c1 & c6, w1 = c1 & ~twos, w6 = c6 & ~twos;
                    sm.A[ai][si] = c1 | c6;
                    if ((c1 | c6) && ai >= 1 && ai <= RT) sm.dirty[cur][ai - 1] = 1u;
                    sm.K[0][ai][si] = w1;
                    sm.K[1][ai][si] = w6;
                    sm.K[2][ai][si] = w6;
                    if (w1) grant(sm, cur, ai - 1, si, 1, w1);
                    if (w6) grant(sm, cur, ai - 1, si, 6, w6);
                    if (twos) enqueue<FLAT>(sm, &sm.qc[cur][1], u, twos);
                    continue;
                }
                uint32_t C[8];
                claims(sm, ai, si, C);
                uint32_t ones = 0u, twos = 0u;
    #pragma unroll
                for (int q = 0; q < 8; ++q) {
                    twos |= ones & C[q];
                    ones |= C[q];
                }
                uint32_t win[8];
    #pragma unroll
                for (int q = 0; q < 8; ++q) win[q] = C[q] & ~twos;
                sm.A[ai][si] = ones;
                if (ones && ai >= 1 && ai <= RT) sm.dirty[cur][ai - 1] = 1u;
                sm.K[0][ai][si] = win[1] | win[3] | win[5] | win[7];
                sm.K[1][ai][si] = win[2] | win[3] | win[6] | win[7];
                sm.K[2][ai][si] = win[4] | win[5] | win[6] | win[7];
    #pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (win[q]) grant(sm, cur, ai - 1, si, q, win[q]);
                if (twos) enqueue<FLAT>(sm, &sm.qc[cur][1], u, twos);
            }
            __syncthreads();
            if (const uint32_t nq = sm.qc[cur][1] & 0xFFFFu) {
                const uint32_t ne = sm.qc[cur][1] >> 16;
                for (uint32_t e = threadIdx.x; e < nq; e += NT) {
                    int u, j;
                    list_entry<FLAT>(sm, ne, nq, e, u, j);
                    const int ai = u / SS, si = u - ai * SS;
                    set_winner(sm, cur, ai, si, j, draw_winner(a, sm, ai, si, j, r0, c0, seed, step));
                }
                __syncthreads();
            }
        }

#else
        // Diagnostic build: no agent logic, every segment takes
        // the no-movement path, i.e. the staged planes + the pheromone stream.
        for (int u = threadIdx.x; u < AROWS * SS; u += NT) (&sm.A[0][0])[u] = 0u;
        __syncthreads();
#endif
        // ------------------------------------------------------------ S3
#ifndef PF_BITS_STREAM_ONLY
        if (!has_agents) {  // (large LEM grids) an empty window: the tile's planes are copied as they are
            // 16-byte segment pairs: NS, the row pitch and the strip offsets are even.
            static_assert(NS % 2 == 0, "strips are whole 16-byte units");
            for (int i = threadIdx.x; i < RT * NS / 2; i += NT) {
                const int rr = i / (NS / 2), sp = i - rr * (NS / 2);
                if (r0 + rr < a.rows_owned)
                    reinterpret_cast<uint4*>(oout + size_t(kGhost + r0 + rr) * a.p.wsp)[sp] =
                        reinterpret_cast<const uint4*>(&sm.pl[slot(base, rr + 3)][2])[sp];
            }
        } else
#endif
        for (int rr = warp; rr < RT; rr += NW) {
            const int lr = r0 + rr;
            if (lr >= a.rows_owned) break;
            const int b = kGhost + lr;
            const int grow = a.row_begin + lr;
            const int rs = slot(base, rr + 3), ai = rr + 1;
            uint2* const orow = oout + size_t(b) * a.p.wsp;
            if (!sm.dirty[cur][rr]) {
                // Nothing arrives or leaves in this row: its planes are copied
                // (and for ACO its pheromone only evaporates).
                if (lane < NS) orow[lane] = sm.pl[rs][lane + 2];
                if (ACO) {
                    const size_t r0c = size_t(b) * W + c0 + lane;
                    TV tc[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s)
                        tc[s] = (c0 + 32 * s + lane < W) ? tin[r0c + 32 * s] : Tau<TV>::make(0.0, 0.0);
#pragma unroll
                    for (int s = 0; s < NS; ++s)
                        if (c0 + 32 * s + lane < W)
                            tout[r0c + 32 * s] = evaporated(tc[s], a.k.factor);
                }
                continue;
            }
            const size_t row0 = size_t(b) * W + c0 + lane;  // this lane's cell in segment 1
            // ACO: issue the whole row's pheromone loads before using any of them
            // (and before the arrival-source fetch, so both round trips overlap).
            TV tv[NS];
            if (ACO) {
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    tv[s] = (c0 + 32 * s + lane < W) ? tin[row0 + 32 * s] : Tau<TV>::make(0.0, 0.0);
            }
            if constexpr (COMPACT) {
                // The row's arrivals, compacted: arrival e (column order) is lane
                // e % 32's, so the per-arrival work (crossing, counters, tour,
                // deposit) runs once per 32 arrivals instead of once per moving
                // segment. alist[e]: its column in the strip | its direction code
                // (row-major, from the winner planes) << 12. The sources of all
                // of them are fetched at once (cp.async, one round trip per row)
                // into asw[e] (word) / atr[e] (ACO tour, then the deposit q / tour);
                // the segment pass below finds arrival e of a cell as the
                // segment's first arrival + the arrivals to its left.
                // Each source is occupied at step start and each destination empty
                // at step start, so no other thread reads or writes these words.
                uint16_t* const alist = sm.alist[warp];
                uint32_t* const asw = &sm.asw[warp][0][0];
                double* const atr = ACO ? &sm.atr[warp][0][0] : nullptr;
                const uint32_t lt = (1u << lane) - 1u;
                uint32_t na = 0;
    #pragma unroll
                for (int si = 1; si <= NS; ++si) {
                    const uint32_t Am = sm.A[ai][si];
                    if (bit(Am, lane)) alist[na + __popc(Am & lt)] = uint16_t(32 * (si - 1) + lane);
                    na += __popc(Am);
                }
                __syncwarp();
                for (uint32_t e = lane; e < na; e += 32) {
                    // The direction code, once per arrival (not per segment and lane),
                    // kept in the entry for the process loop.
                    const int cc = alist[e], si = (cc >> 5) + 1, j = cc & 31;
                    const int kc = int(bit(sm.K[0][ai][si], j) | bit(sm.K[1][ai][si], j) << 1 | bit(sm.K[2][ai][si], j) << 2);
                    alist[e] = uint16_t(kc << 12 | cc);
                    const size_t src = size_t(b + kDR[kc]) * W + (c0 + cc + kDC[kc]);
                    cp_async<4>(asw + e, cw + src);
                    if (ACO) cp_async<8>(atr + e, tour + src);
                }
                cp_async_wait_all();
                __syncwarp();
                for (uint32_t e = lane; e < na; e += 32) {
                    const int cc = alist[e] & 0xFFF, kc = alist[e] >> 12;
                    const uint32_t sw = asw[e];
                    const uint32_t group = sw >> 30;
                    uint32_t nw = sw;
                    if (!(sw & kCrossedBit) && crossed_at(group, grow, a.k.H, band)) {  // src/engine.cpp:163-170
                        nw |= kCrossedBit;
                        if (group == 1u) ++ntop;
                        else ++nbot;
                    }
                    ++moved;
                    const size_t gi = size_t(b) * W + c0 + cc;
                    cw[gi] = nw;
                    if (ACO) {  // tour += 1 or sqrt(2) (src/engine.cpp:159-160); deposit q / tour (src/aco.cpp:119-123)
                        const double tour_new = __dadd_rn(atr[e], is_diag(kc) ? a.k.diag : 1.0);
                        tour[gi] = tour_new;
                        atr[e] = __ddiv_rn(a.k.q, tour_new);
                    }
                }
                __syncwarp();
                uint2 mine = make_uint2(kWall, kWall);
                uint32_t e0 = 0;  // arrivals in the segments left of si
    #pragma unroll
                for (int si = 1; si <= NS; ++si) {
                    const int gc = c0 + 32 * (si - 1) + lane;
                    const bool valid = gc < W;
                    const uint32_t Am = sm.A[ai][si], Gm = sm.G[cur][rr][si];
                    uint2 np = sm.pl[rs][si + 1];
                    const size_t gi = row0 + 32 * (si - 1);
                    const uint32_t ea = e0 + __popc(Am & lt);
                    e0 += __popc(Am);
                    if ((Am | Gm) == 0u) {  // warp-uniform: nothing moves in this segment
                        if (ACO && valid) {
                            tout[gi] = evaporated(tv[si - 1], a.k.factor);
                        }
                    } else {
                        const bool arrived = bit(Am, lane) != 0u;
                        const uint32_t group = arrived ? asw[ea] >> 30 : 0u;
                        const uint32_t top = __ballot_sync(0xFFFFFFFFu, group == 1u);
                        np.x = (np.x & ~Gm) | top;  // vacated sources clear, arrivals set
                        np.y = (np.y & ~Gm) | (Am & ~top);
                        if (ACO && valid) {  // evaporate, then deposit (src/engine.cpp:124-131, src/aco.cpp:119-123)
                            double tx = __dmul_rn(double(tv[si - 1].x), a.k.factor);
                            double ty = __dmul_rn(double(tv[si - 1].y), a.k.factor);
                            if (arrived) {
                                const double dep = atr[ea];
                                if (group == 1u) tx = __dadd_rn(tx, dep);
                                else ty = __dadd_rn(ty, dep);
                            }
                            tout[gi] = Tau<TV>::make(tx, ty);
                        }
                    }
                    if (lane == si - 1) mine = np;
                }
                if (lane < NS) orow[lane] = mine;
            } else {
                // Sparse arrivals (large grids): per segment, lane = column.
                // The sources of this row's arrivals: all their loads are in
                // flight together (one round trip per row, not one per segment).
                // Each source is occupied at step start, so nothing writes it.
    #pragma unroll
                for (int si = 1; si <= NS; ++si) {
                    if (bit(sm.A[ai][si], lane)) {
                        const int kc = int(bit(sm.K[0][ai][si], lane) | bit(sm.K[1][ai][si], lane) << 1 |
                                           bit(sm.K[2][ai][si], lane) << 2);
                        const size_t src = size_t(b + kDR[kc]) * W + (c0 + 32 * (si - 1) + lane + kDC[kc]);
                        cp_async<4>(&sm.asw[warp][si - 1][lane], cw + src);
                        if (ACO) cp_async<8>(&sm.atr[warp][si - 1][lane], tour + src);
                    }
                }
                cp_async_wait_all();
                __syncwarp();
                uint2 mine = make_uint2(kWall, kWall);
    #pragma unroll
                for (int si = 1; si <= NS; ++si) {
                    const int gc = c0 + 32 * (si - 1) + lane;
                    const bool valid = gc < W;
                    const uint32_t Am = sm.A[ai][si], Gm = sm.G[cur][rr][si];
                    uint2 np = sm.pl[rs][si + 1];
                    const size_t gi = row0 + 32 * (si - 1);
                    if ((Am | Gm) == 0u) {  // warp-uniform: nothing moves in this segment
                        if (ACO && valid) {
                            tout[gi] = evaporated(tv[si - 1], a.k.factor);
                        }
                    } else {
                        const bool arrived = bit(Am, lane) != 0u;
                        uint32_t group = 0;
                        double tour_new = 0.0;
                        if (arrived) {
                            const int kc = int(bit(sm.K[0][ai][si], lane) | bit(sm.K[1][ai][si], lane) << 1 |
                                               bit(sm.K[2][ai][si], lane) << 2);
                            const uint32_t sw = sm.asw[warp][si - 1][lane];
                            group = sw >> 30;
                            uint32_t nw = sw;
                            if (!(sw & kCrossedBit) && crossed_at(group, grow, a.k.H, band)) {  // src/engine.cpp:163-170
                                nw |= kCrossedBit;
                                if (group == 1u) ++ntop;
                                else ++nbot;
                            }
                            ++moved;
                            cw[gi] = nw;  // empty at step start: nobody reads it this step
                            if (ACO) {    // tour += 1 or sqrt(2) (src/engine.cpp:159-160)
                                tour_new = __dadd_rn(sm.atr[warp][si - 1][lane], is_diag(kc) ? a.k.diag : 1.0);
                                tour[gi] = tour_new;
                            }

                        }
                        const uint32_t top = __ballot_sync(0xFFFFFFFFu, group == 1u);
                        const uint32_t bot = __ballot_sync(0xFFFFFFFFu, group == 2u);
                        np.x = (np.x & ~Gm) | top;  // vacated sources clear, arrivals set
                        np.y = (np.y & ~Gm) | bot;
                        if (ACO && valid) {  // evaporate, then deposit (src/engine.cpp:124-131, src/aco.cpp:119-123)
                            double tx = __dmul_rn(double(tv[si - 1].x), a.k.factor);
                            double ty = __dmul_rn(double(tv[si - 1].y), a.k.factor);
                            if (arrived) {
                                const double dep = __ddiv_rn(a.k.q, tour_new);
                                if (group == 1u) tx = __dadd_rn(tx, dep);
                                else ty = __dadd_rn(ty, dep);
                            }
                            tout[gi] = Tau<TV>::make(tx, ty);
                        }
                    }
                    if (lane == si - 1) mine = np;
                }
                if (lane < NS) orow[lane] = mine;
            }
        }
        __syncthreads();  // end of tile: the window's slots may be refilled
        if (MIRROR && (r0 < kGhost || r0 + RT > a.rows_owned - kGhost)) mirror_tile<ACO, TV>(a, par, rep, it.strip, r0);
        base = slot(base, RT);
        cur ^= 1;
    }
    base = next_base;
    // Counters of this item go to its replica's StepReport (src/engine.cpp:172-174).
    moved = __reduce_add_sync(0xFFFFFFFFu, moved);
    ntop = __reduce_add_sync(0xFFFFFFFFu, ntop);
    nbot = __reduce_add_sync(0xFFFFFFFFu, nbot);
    if (lane == 0 && (moved | ntop | nbot)) {
        atomicAdd(&sm.cnt[0], moved);
        atomicAdd(&sm.cnt[1], ntop);
        atomicAdd(&sm.cnt[2], nbot);
    }
    moved = ntop = nbot = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* rep_slot = a.reports + (size_t(rep) * a.report_cap + step % uint32_t(a.report_cap)) * 4;
        if (it.strip == 0 && it.chunk == 0) rep_slot[0] = step;
        if (sm.cnt[0]) atomicAdd(&rep_slot[1], sm.cnt[0]);
        if (sm.cnt[1]) atomicAdd(&rep_slot[2], sm.cnt[1]);
        if (sm.cnt[2]) atomicAdd(&rep_slot[3], sm.cnt[2]);
        sm.cnt[0] = sm.cnt[1] = sm.cnt[2] = 0u;
        if (MIRROR && it.sides) signal_boundary(a, it.sides, step, strips, n_chunks, n_tiles);  // after the barrier: all mirror stores fenced
        // Release the item's tiles. The barrier above orders every thread's
        // stores of the item before this thread's; the gpu-scope release
        // (cumulative) publishes them with the flag (as CUTLASS's semaphore).
        if (multi) {
            for (int t = it.t_first; t < it.t_end; ++t) {
                uint32_t* f = a.tile_done + (size_t(rep) * strips + it.strip) * n_tiles + t;
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(step + 1u) : "memory");
            }
        }
    }
    item = sm.item[ipar];  // claimed during the last tile (visible after its barriers)
    islot = ipar;
    ipar ^= 1;
    if ((!kCrossPrefetch || (multi && sm.defer[islot])) && item < n_all) {
        // Small ring, or a deferred multi-step item: the next item's window
        // is loaded only now, into the slots the finished item released.
        if (warp == kIoWarp) {
            const Item nit = read_item(sm.idec[islot], n_tiles, a.tiles_per_cta);
            if (MIRROR && nit.sides && lane == 0) wait_boundary(a, nit.sides, step0);
            if (multi && nit.sl > 0) deps_ready(a, nit, step0 + uint32_t(nit.sl), strips, n_tiles, true);
            __syncwarp();
            load_rows(sm, a, parity ^ (nit.sl & 1), nit, nit.t_first * RT, base, 0, SR, &sm.mbar[nload & 1]);
        }
        __syncthreads();  // wall rows written by the I/O warp are visible to all
    }
    if (item < n_all) ++nload;
    }  // work items
}

// CTAs per SM: the register budget (kRegCtas), capped by shared memory (1 KB
// reserved per CTA); one fewer (more registers) for large ACO grids.
constexpr int smem_ctas(bool aco) { return int((228 * 1024) / (kSmemBytes[aco ? 1 : 0] + 1024)); }
constexpr int kCtasLem = kRegCtas < smem_ctas(false) ? kRegCtas : smem_ctas(false);
constexpr int kCtasDefault = kRegCtas < smem_ctas(true) ? kRegCtas : smem_ctas(true);
constexpr int kCtasHbm = kCtasDefault > 1 && NT == 256 ? 3 : kCtasDefault;
// Large LEM grids: 5 CTAs (48 registers, small spills) hide more of the
// issue-bound bit logic (C5 LEM -5.5%); smaller batched grids keep 4 (C3 x64
// +2% with 5).
constexpr int kCtasLemBig = NT == 256 && smem_ctas(false) >= 5 ? 5 : kCtasLem;
static_assert(kCtasLem >= 1 && kCtasDefault >= 1, "shared memory must fit one CTA per SM");

template <class TV>
int configure_aco(int bytes) {
    for (auto f : {step_bits_kernel<true, kCtasDefault, false, true, false, TV>,
                   step_bits_kernel<true, kCtasHbm, false, false, false, TV>,
                   step_bits_kernel<true, kCtasDefault, true, true, false, TV>,
                   step_bits_kernel<true, kCtasHbm, true, false, false, TV>,
                   step_bits_kernel<true, kCtasDefault, false, true, true, TV>})
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return 1;
    return 0;
}

int configure() {
    const int lem = int(kSmemBytes[0]), aco = int(kSmemBytes[1]);
    for (auto f : {step_bits_kernel<false, kCtasLem, false, true, false>, step_bits_kernel<false, kCtasLem, true, true, false>,
                   step_bits_kernel<false, kCtasLem, false, true, true>,
                   step_bits_kernel<false, kCtasLemBig, false, false, false>, step_bits_kernel<false, kCtasLemBig, true, false, false>})
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, lem) != cudaSuccess) return 1;
    if (configure_aco<double2>(aco) || configure_aco<float2>(aco)) return 1;
    return 0;
}

// Launch with programmatic stream serialization (PDL): the next step's
// kernel may be scheduled while this one finishes its last items.
template <class Kernel>
static void launch_pdl(Kernel kernel, dim3 grid, size_t smem, cudaStream_t s, const StepArgs& b, int slot_idx,
                       int parity) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, b, slot_idx, parity);
}

template <class TV>
static void launch_aco(const StepArgs& b, bool hbm, bool mirror, dim3 grid, size_t bytes, cudaStream_t s, int slot_idx,
                       int parity) {
    if (hbm) {
        if (mirror) launch_pdl(step_bits_kernel<true, kCtasHbm, true, false, false, TV>, grid, bytes, s, b, slot_idx, parity);
        else launch_pdl(step_bits_kernel<true, kCtasHbm, false, false, false, TV>, grid, bytes, s, b, slot_idx, parity);
    } else {
        if (mirror) launch_pdl(step_bits_kernel<true, kCtasDefault, true, true, false, TV>, grid, bytes, s, b, slot_idx, parity);
        else if (b.nsteps > 1) launch_pdl(step_bits_kernel<true, kCtasDefault, false, true, true, TV>, grid, bytes, s, b, slot_idx, parity);
        else launch_pdl(step_bits_kernel<true, kCtasDefault, false, true, false, TV>, grid, bytes, s, b, slot_idx, parity);
    }
}

#ifndef PF_MULTI_MAX_ITEMS_PER_CTA
#define PF_MULTI_MAX_ITEMS_PER_CTA 16  // x128 batches (13 per CTA) -1.7% multi-step, x256 (26) +2%
#endif

// Persistent grid: one CTA per resident slot (SMs x 3, 4 or 5) at most. Work
// items are chunks of up to 16 consecutive RT-row tiles of one strip of one
// replica, about items_per_cta items per CTA (pf_context.cu: one tile per
// item for ACO, two for C5 LEM; a short tail at the end of the step).
int launch(const StepArgs& a, int slot_idx, int parity, cudaStream_t s) {
    const int strips = (a.k.W + NS * 32 - 1) / (NS * 32);
    const int n_tiles = (a.rows_owned + RT - 1) / RT;
    const bool aco = a.k.model == 1;
    const bool big = double(a.k.W) * a.rows_buf >= double(1 << 22);  // >= 4M cells per replica
    const bool hbm = aco && big;
    const int ctas = !aco ? (big ? kCtasLemBig : kCtasLem) : (hbm ? kCtasHbm : kCtasDefault);
    // A linked neighbour on the same GPU (tests, development) needs resident
    // slots for its own boundary items while ours wait for them in-kernel:
    // take at most half of them. (One shard per GPU never shares.)
    const long long ctas_max = (long long)a.num_sms * ctas / (a.peer_same_device ? 2 : 1);
    const long long tiles = (long long)strips * n_tiles * a.replicas;
    StepArgs b = a;
    b.tiles_per_cta = int(std::max<long long>(1, std::min<long long>(16, tiles / (ctas_max * a.items_per_cta))));
    const long long items = (long long)strips * ((n_tiles + b.tiles_per_cta - 1) / b.tiles_per_cta) * a.replicas;
    const bool mirror = a.peer[0].cell || a.peer[1].cell;  // linked shard: fused halo exchange
    // Multi-step launches pay where a step's tail is a large part of it: a
    // few items per resident CTA (the 480^2 x64 batches: C4 -9%, C3 -10%; x128 -1.7%).
    // With many items per CTA (C5) the tail is negligible and the per-item
    // dependency polls cost (C5 LEM +11%); with fewer items than CTAs
    // (single 480^2 scenarios) the flag round trips cost more than the
    // launches they replace (C1 +25%). Those take one launch per step.
    if (b.nsteps > 1 && (mirror || big || items < ctas_max || items > PF_MULTI_MAX_ITEMS_PER_CTA * ctas_max)) {
        const int n = b.nsteps;
        b.nsteps = 1;
        int launches = 0;
        for (int i = 0; i < n; ++i) launches += launch(b, slot_idx + i, parity ^ (i & 1), s);
        return launches;
    }
    dim3 grid(unsigned(std::min(items * std::max(1, b.nsteps), ctas_max)));
    const size_t bytes = kSmemBytes[aco ? 1 : 0];
    if (!aco && big) {
        if (mirror) launch_pdl(step_bits_kernel<false, kCtasLemBig, true, false, false>, grid, bytes, s, b, slot_idx, parity);
        else launch_pdl(step_bits_kernel<false, kCtasLemBig, false, false, false>, grid, bytes, s, b, slot_idx, parity);
    } else if (!aco) {
        if (mirror) launch_pdl(step_bits_kernel<false, kCtasLem, true, true, false>, grid, bytes, s, b, slot_idx, parity);
        else if (b.nsteps > 1) launch_pdl(step_bits_kernel<false, kCtasLem, false, true, true>, grid, bytes, s, b, slot_idx, parity);
        else launch_pdl(step_bits_kernel<false, kCtasLem, false, true, false>, grid, bytes, s, b, slot_idx, parity);
    } else if (b.tau_f32) {  // (large grids: 3 CTAs/SM as for fp64; 4 measured 7.5% slower at C5)
        launch_aco<float2>(b, hbm, mirror, grid, bytes, s, slot_idx, parity);
    } else {
        launch_aco<double2>(b, hbm, mirror, grid, bytes, s, slot_idx, parity);
    }
    return 1;
}

}  // namespace PF_BITS_NAMESPACE
}  // namespace pfk
