// Bit-sliced fused step kernel (the default product path, PF_KERNEL_FUSED).
//
// The per-step update (StepEngine::step, src/engine.cpp:53-193) is evaluated
// on 32-cell row segments held as 32-bit masks, so the common work costs one
// ALU op per 32 cells; only agents that must draw (forward blocked, some slot
// open) and destinations with >= 2 claimants fall to per-cell scalar code, and
// those are compacted into shared-memory work lists so every lane takes one.
//
// Persistent column sweep: a CTA owns a strip of NS 32-column segments and a
// run of consecutive RT-row tiles. The step-start cell words of the strip live
// in a shared-memory ring of staged rows (tile + 3-row halo + the next tile's
// rows); while a tile is processed, TMA bulk copies (cp.async.bulk +
// mbarrier) bring the next tile's RT new rows, so every row is loaded and
// balloted once and the load latency hides behind the compute.
//
//   S0 stage   ballot the new rows into occupancy planes v30 / v31 (bits 30/31
//              of the word: Top = v30 & ~v31, Bottom = v31 & ~v30,
//              Empty = ~(v30 | v31)).
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
//   S3 commit  warp per segment-row, lane = column: new cell word (arrival /
//              vacate / unchanged), crossing + counters, ACO evaporation +
//              deposit and tour (src/engine.cpp:124-175).
#include <algorithm>

#include "pf_internal.h"

namespace pfk {

using namespace pfdev;

namespace {

constexpr int RT = 16;           // output rows per tile
constexpr int NS = 8;            // output 32-column segments per strip
constexpr int SR = RT + 6;       // staged rows of one tile: -3 .. RT+2
#ifndef PF_BITS_RING
#define PF_BITS_RING (2 * SR)
#endif
// Ring slots: the current window + the next tile's rows, or (2 * SR) the next
// item's whole window, prefetched during an item's last tile.
constexpr int RING = PF_BITS_RING;
constexpr bool kCrossPrefetch = RING >= 2 * SR;
static_assert(RING >= SR + RT, "the ring must hold a window and the next tile's rows");
constexpr int SS = NS + 2;       // staged segments: -1 .. NS
// Staged columns: the strip plus a 4-column halo on each side (the dependency
// radius is 3; 4 keeps TMA rows 16-byte aligned). Bit j of plane segment si
// (si = 0 .. NS+1, segment si-1 of the strip) is staged column
// 32 * si + j - WOFF; the halo segments 0 and NS+1 only have bits 28..31 and
// 0..3 staged.
constexpr int HALO = 4;
constexpr int SW = NS * 32 + 2 * HALO;
constexpr int WOFF = 32 - HALO;
constexpr int NT = 256;          // threads per CTA
constexpr int NW = NT / 32;
constexpr int DROWS = RT + 4;    // intent rows -2 .. RT+1
constexpr int AROWS = RT + 2;    // resolution rows -1 .. RT
constexpr int NU = DROWS * SS;   // intent units (>= resolution units AROWS * SS)
static_assert(NU * 32 < (1 << 16), "work-list bit counts must fit 16 bits");

struct Smem {
    uint32_t word[RING][SW];  // rows are 1,056 B: every row start is 16-byte aligned for TMA
    uint32_t v30[RING][SS];
    uint32_t v31[RING][SS];
    uint32_t D[8][DROWS][SS];
    uint32_t A[AROWS][SS];
    uint32_t K[3][AROWS][SS];
    uint32_t G[RT][SS];
    uint32_t dirty[RT];  // owned row has an arrival or a vacate
    // Scalar work list (S1 draws, then reused for S2 contested cells): one
    // entry per unit with work, in the order a packed counter handed out
    // (entry count << 16 | bit count, one native 32-bit shared atomic; at
    // most NU * 32 < 2^16 bits), so qp (first rank of the entry) is sorted
    // and rank r maps to its (unit, bit) by binary search. Bounded by the
    // unit count: it cannot overflow.
    uint32_t qu[NU];  // unit
    uint32_t qm[NU];  // its bits
    uint32_t qp[NU];  // rank of its first bit
    unsigned long long mbar[2];
    uint32_t qc[2];  // [0] S1 draws, [1] S2 contested cells
    int item;
    uint32_t cnt[3];
};

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

// Ring slot of staged row sr (0 = tile row -3) for a window starting at base.
__device__ __forceinline__ int slot(int base, int sr) {
    const int s = base + sr;
    return s >= RING ? s - RING : s;
}

// Emptiness around one intent unit: the eight neighbour planes, shifted so
// bit j is the neighbour of column j.
struct Around {
    uint32_t em, emL, emR, e0L, e0R, ep, epL, epR;
};

__device__ __forceinline__ Around around(const Smem& sm, int base, int sr, int si) {
    const int rm = slot(base, sr - 1), r0 = slot(base, sr), rp = slot(base, sr + 1);
    auto E = [&](int row, int seg) -> uint32_t {
        return (seg < 0 || seg >= SS) ? 0u : ~(sm.v30[row][seg] | sm.v31[row][seg]);
    };
    Around n;
    n.em = E(rm, si);
    n.ep = E(rp, si);
    const uint32_t e0 = E(r0, si);
    n.emL = from_left(n.em, E(rm, si - 1));
    n.emR = from_right(n.em, E(rm, si + 1));
    n.e0L = from_left(e0, E(r0, si - 1));
    n.e0R = from_right(e0, E(r0, si + 1));
    n.epL = from_left(n.ep, E(rp, si - 1));
    n.epR = from_right(n.ep, E(rp, si + 1));
    return n;
}

// Claims on the destinations of resolution unit (row ai-1, segment si).
__device__ __forceinline__ void claims(const Smem& sm, int ai, int si, uint32_t (&C)[8]) {
    auto D = [&](int k, int row, int seg) -> uint32_t { return (seg < 0 || seg >= SS) ? 0u : sm.D[k][row][seg]; };
    const int dm = ai, d0 = ai + 1, dp = ai + 2;  // intent rows of rr-1, rr, rr+1
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
__device__ __forceinline__ void grant(Smem& sm, int rr, int si, int k, uint32_t wk) {
    const int g = rr + kDR[k];
    if (g < 0 || g >= RT) return;
    sm.dirty[g] = 1u;
    const int dc = kDC[k];
    if (dc == 0) {
        atomicOr(&sm.G[g][si], wk);
    } else if (dc < 0) {
        atomicOr(&sm.G[g][si], wk >> 1);
        if ((wk & 1u) && si > 0) atomicOr(&sm.G[g][si - 1], 0x80000000u);
    } else {
        atomicOr(&sm.G[g][si], wk << 1);
        if ((wk >> 31) && si + 1 < SS) atomicOr(&sm.G[g][si + 1], 1u);
    }
}

// Add unit u's bits `mask` to work list `list`.
__device__ __forceinline__ void enqueue(Smem& sm, int u, uint32_t mask, int list) {
    const uint32_t old = atomicAdd(&sm.qc[list], (1u << 16) | uint32_t(__popc(mask)));
    const int e = int(old >> 16);
    sm.qu[e] = uint32_t(u);
    sm.qm[e] = mask;
    sm.qp[e] = old & 0xFFFFu;
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

// Work-list rank r -> (unit, bit), n entries.
__device__ __forceinline__ void list_entry(const Smem& sm, uint32_t n, uint32_t r, int& u, int& j) {
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
// lem_select / aco_select (src/lem.cpp:28-60, src/aco.cpp:64-92).
template <bool ACO>
__device__ __forceinline__ int draw_intent(const StepArgs& a, const Smem& sm, int base,
                                           const double2* __restrict__ tin, int di, int si, int j, bool bottom,
                                           int r0, int c0, uint64_t seed, uint32_t step) {
    const int sr = di + 1;
    const Around n = around(sm, base, sr, si);
    uint32_t open;  // goal-relative slots F FL FR L R B BL BR
    if (!bottom)
        open = bit(n.ep, j) | bit(n.epL, j) << 1 | bit(n.epR, j) << 2 | bit(n.e0L, j) << 3 | bit(n.e0R, j) << 4 |
               bit(n.em, j) << 5 | bit(n.emL, j) << 6 | bit(n.emR, j) << 7;
    else
        open = bit(n.em, j) | bit(n.emR, j) << 1 | bit(n.emL, j) << 2 | bit(n.e0R, j) << 3 | bit(n.e0L, j) << 4 |
               bit(n.ep, j) << 5 | bit(n.epR, j) << 6 | bit(n.epL, j) << 7;
    const uint32_t id = sm.word[slot(base, sr)][si * 32 + j - WOFF] & kIdMask;
    int s;
    if (!ACO) {
        s = lem_choose(a.kc, open, seed, step, id);
    } else {
        const int W = a.k.W;
        const int b = kGhost + r0 + di - 2;
        const int c = c0 + 32 * (si - 1) + j;
        // All eight neighbour loads are issued before any is used (they are
        // in bounds for every agent cell: rows b-1 .. b+1 lie inside the
        // buffer and a column step off the row lands in the adjacent row).
        const double* t0 = reinterpret_cast<const double*>(tin + size_t(b) * W + c) + (bottom ? 1 : 0);
        double tn[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint8_t code = bottom ? uint8_t(7 - kSlotCodeTop[i]) : kSlotCodeTop[i];
            tn[i] = __ldg(t0 + 2 * (ptrdiff_t(kDR[code]) * W + kDC[code]));
        }
        double num[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            num[i] = (open >> i & 1u) ? __dmul_rn(pheromone_term(a.kc, tn[i]), __ldg(&a.kc->eta[i])) : 0.0;
        s = aco_choose(num, open, seed, step, id);
    }
    return bottom ? 7 - kSlotCodeTop[s] : kSlotCodeTop[s];
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

__device__ __forceinline__ void set_winner(Smem& sm, int ai, int si, int j, int k) {
    const uint32_t b = 1u << j;
    if (k & 1) atomicOr(&sm.K[0][ai][si], b);
    if (k & 2) atomicOr(&sm.K[1][ai][si], b);
    if (k & 4) atomicOr(&sm.K[2][ai][si], b);
    grant(sm, ai - 1, si, k, b);
}

// One work item: a chunk of consecutive RT-row tiles of one strip of one
// replica, with the strip's column window.
struct Item {
    int rep, strip, chunk, c0, t_first, t_end;
    int col_lo, fill_lo, fill_hi;  // arena columns [col_lo, ...) land in staged columns [fill_lo, fill_hi)
};

__device__ __forceinline__ Item decode_item(int item, int strips, int n_chunks, int n_tiles, int tiles_per_item,
                                            int W) {
    Item it;
    it.rep = item / (strips * n_chunks);
    it.strip = (item / n_chunks) % strips;
    it.chunk = item % n_chunks;
    it.c0 = it.strip * (NS * 32);
    it.t_first = it.chunk * tiles_per_item;
    it.t_end = min(it.t_first + tiles_per_item, n_tiles);
    it.col_lo = max(it.c0 - HALO, 0);
    const int col_hi = min(it.c0 + 32 * NS + HALO, W);  // 16-byte aligned: c0 % 256 == 0, W % 16 == 0
    it.fill_lo = it.col_lo - (it.c0 - HALO);
    it.fill_hi = col_hi - (it.c0 - HALO);
    return it;
}

// Issue the TMA loads of `nrows` staged rows (tile rows first_sr.., relative
// to the tile at r0) of item `it` into their ring slots, completing on
// mbarrier m; the strip's columns outside the arena and rows past the end of
// the buffer are written as walls. Called by one full warp.
__device__ __forceinline__ void load_rows(Smem& sm, const StepArgs& a, int parity, const Item& it, int r0, int base,
                                          int first_sr, int nrows, unsigned long long* m) {
    const int lane = threadIdx.x & 31;
    const int W = a.k.W;
    const uint32_t* cin = a.p.cell[parity] + size_t(it.rep) * a.p.plane;
    const int b_first = kGhost + r0 - 3 + first_sr;
    const int nvalid = max(0, min(nrows, a.rows_buf - b_first));
    const int ncols = it.fill_hi - it.fill_lo;
    if (lane == 0) mbar_expect_tx(m, uint32_t(nvalid) * uint32_t(ncols) * 4u);
    __syncwarp();
    for (int i = lane; i < nvalid; i += 32)
        bulk_g2s(&sm.word[slot(base, first_sr + i)][it.fill_lo], cin + size_t(b_first + i) * W + it.col_lo,
                 uint32_t(ncols) * 4u, m);
    const int nfill = SW - ncols;  // wall columns at the arena's left / right edge
    for (int i = lane; i < nvalid * nfill; i += 32) {
        const int r = i / nfill, c = i - r * nfill;
        sm.word[slot(base, first_sr + r)][c < it.fill_lo ? c : it.fill_hi + (c - it.fill_lo)] = kWall;
    }
    for (int i = nvalid; i < nrows; ++i)
        for (int c = lane; c < SW; c += 32) sm.word[slot(base, first_sr + i)][c] = kWall;
}

template <bool ACO>
__global__ void __launch_bounds__(NT, 3) step_bits_kernel(const StepArgs a, int slot_idx, int parity) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    const int W = a.k.W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t step = *a.d_step + uint32_t(slot_idx);
    const int strips = (W + NS * 32 - 1) / (NS * 32);
    const int n_tiles = (a.rows_owned + RT - 1) / RT;
    const int n_chunks = (n_tiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
    const int n_items = strips * n_chunks * a.replicas;
    uint32_t* work = a.work + step % uint32_t(a.report_cap);

    if (threadIdx.x == 0) {
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        fence_mbar_init();
        sm.cnt[0] = sm.cnt[1] = sm.cnt[2] = 0u;
    }
    __syncthreads();
    // Work item = (replica, strip, chunk of tiles_per_cta consecutive tiles),
    // taken from a per-step counter so heavy (crowded) chunks balance out.
    // The next item is claimed during the current item's last tile and its
    // first window is loaded into the other half of the ring meanwhile.
    int item = 0;
    if (warp == 0) {
        if (lane == 0) item = int(atomicAdd(work, 1u));
        item = __shfl_sync(0xFFFFFFFFu, item, 0);
        if (lane == 0) sm.item = item;
        if (item < n_items) {
            const Item first = decode_item(item, strips, n_chunks, n_tiles, a.tiles_per_cta, W);
            load_rows(sm, a, parity, first, first.t_first * RT, 0, 0, SR, &sm.mbar[0]);
        }
    }
    __syncthreads();  // item id and wall rows written by warp 0 are visible to all
    item = sm.item;
    uint32_t moved = 0, ntop = 0, nbot = 0;
    uint32_t nload = item < n_items ? 1u : 0u;  // load i completes mbar[i & 1], phase i >> 1
    int base = 0;                               // ring slot of staged row 0 of the current tile
    while (item < n_items) {
    const Item it = decode_item(item, strips, n_chunks, n_tiles, a.tiles_per_cta, W);
    const int rep = it.rep, c0 = it.c0;
    const uint64_t seed = __ldg(&a.rep[rep].seed);
    const int band = __ldg(&a.rep[rep].band);
    const size_t plane_base = size_t(rep) * a.p.plane;
    uint32_t* __restrict__ cout = a.p.cell[parity ^ 1] + plane_base;
    const double2* __restrict__ tin = ACO ? a.p.tau[parity] + plane_base : nullptr;
    double2* __restrict__ tout = ACO ? a.p.tau[parity ^ 1] + plane_base : nullptr;
    double* __restrict__ tour = ACO ? a.p.tour + plane_base : nullptr;
    int next_base = 0;

    for (int t = it.t_first; t < it.t_end; ++t) {
        const int k = t - it.t_first;  // tile index within the item (k == 0: full window)
        const int r0 = t * RT;         // owned-local row of the tile
        const uint32_t my_load = nload - 1;  // the load that brought this tile's new rows
        // Prefetch into the half of the ring this tile does not use (its
        // previous readers all passed the end-of-tile barrier): the next
        // tile's RT new rows, or on the last tile the next item's window.
        if (t + 1 < it.t_end) {
            if (warp == 0) load_rows(sm, a, parity, it, r0 + RT, slot(base, RT), 6, RT, &sm.mbar[nload & 1]);
            ++nload;
        } else {
            next_base = kCrossPrefetch ? slot(base, SR) : 0;
            if (warp == 0) {
                int nx = 0;
                if (lane == 0) nx = int(atomicAdd(work, 1u));
                nx = __shfl_sync(0xFFFFFFFFu, nx, 0);
                if (lane == 0) sm.item = nx;
                if (kCrossPrefetch && nx < n_items) {
                    const Item nit = decode_item(nx, strips, n_chunks, n_tiles, a.tiles_per_cta, W);
                    load_rows(sm, a, parity, nit, nit.t_first * RT, next_base, 0, SR, &sm.mbar[nload & 1]);
                }
            }
        }
        for (int i = threadIdx.x; i < RT * SS; i += NT) (&sm.G[0][0])[i] = 0u;
        if (threadIdx.x < RT) sm.dirty[threadIdx.x] = 0u;
        if (threadIdx.x == 0) sm.qc[0] = sm.qc[1] = 0u;
        mbar_wait(&sm.mbar[my_load & 1], (my_load >> 1) & 1u);

        // ------------------------------------------------------------ S0
        // Thread per new segment-row: eight 16-byte shared loads (chunk order
        // rotated by lane, so a quarter-warp hits eight distinct bank groups),
        // the top byte of each word packed with PRMT, bits 31 / 30 of four
        // words gathered into a nibble by one multiply.
        {
            const int first = k == 0 ? 0 : 6;
            for (int u = threadIdx.x; u < (SR - first) * SS; u += NT) {
                const int sr = first + u / SS, si = u % SS;
                const int rs = slot(base, sr);
                auto nibbles = [](const uint4& q, uint32_t& n30, uint32_t& n31) {
                    const uint32_t top =
                        __byte_perm(__byte_perm(q.x, q.y, 0x0073), __byte_perm(q.z, q.w, 0x0073), 0x5410);
                    n31 = ((top & 0x80808080u) * 0x00204081u) >> 28;
                    n30 = (((top & 0x40404040u) * 0x00204081u) >> 27) & 0xFu;
                };
                uint32_t v30 = 0u, v31 = 0u;
                if (si == 0 || si == SS - 1) {  // halo segment: 4 staged columns, the rest walls
                    const bool left = si == 0;
                    uint32_t n30, n31;
                    nibbles(*reinterpret_cast<const uint4*>(&sm.word[rs][left ? 0 : SW - HALO]), n30, n31);
                    v30 = left ? (0x0FFFFFFFu | n30 << 28) : (0xFFFFFFF0u | n30);
                    v31 = left ? (0x0FFFFFFFu | n31 << 28) : (0xFFFFFFF0u | n31);
                } else {
                    const uint4* p = reinterpret_cast<const uint4*>(&sm.word[rs][si * 32 - WOFF]);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int c = (i + lane) & 7;
                        uint32_t n30, n31;
                        nibbles(p[c], n30, n31);
                        v31 |= n31 << (4 * c);
                        v30 |= n30 << (4 * c);
                    }
                }
                sm.v30[rs][si] = v30;
                sm.v31[rs][si] = v31;
            }
        }
        __syncthreads();

        // ------------------------------------------------------------ S1
        // Intents for rows -2 .. RT+1, all staged segments (halo segments
        // only at the two columns next to the strip).
        for (int u = threadIdx.x; u < DROWS * SS; u += NT) {
            const int di = u / SS, si = u - di * SS;  // di = rr + 2
            const int rs = slot(base, di + 1);
            const Around n = around(sm, base, di + 1, si);
            const uint32_t v30 = sm.v30[rs][si], v31 = sm.v31[rs][si];
            const uint32_t segmask = si == 0 ? 0xC0000000u : (si == SS - 1 ? 0x00000003u : 0xFFFFFFFFu);
            const uint32_t T = v30 & ~v31 & segmask, B = v31 & ~v30 & segmask;
            uint32_t d[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) d[q] = 0u;
            d[6] = T & n.ep;  // Top forward: (+1, 0)
            d[1] = B & n.em;  // Bottom forward: (-1, 0)
            const uint32_t any8 = n.ep | n.epL | n.epR | n.e0L | n.e0R | n.em | n.emL | n.emR;
            const uint32_t slow = ((T & ~n.ep) | (B & ~n.em)) & any8;
            if (slow) enqueue(sm, u, slow, 0);
#pragma unroll
            for (int q = 0; q < 8; ++q) sm.D[q][di][si] = d[q];
        }
        __syncthreads();
        // Draws, spread evenly over the CTA (the barrier is skipped,
        // uniformly, when there are none).
        if (const uint32_t nq = sm.qc[0] & 0xFFFFu) {
            const uint32_t ne = sm.qc[0] >> 16;
            for (uint32_t e = threadIdx.x; e < nq; e += NT) {
                int u, j;
                list_entry(sm, ne, e, u, j);
                const int di = u / SS, si = u - di * SS;
                const bool bottom = bit(sm.v31[slot(base, di + 1)][si], j) != 0u;
                const int code = draw_intent<ACO>(a, sm, base, tin, di, si, j, bottom, r0, c0, seed, step);
                atomicOr(&sm.D[code][di][si], 1u << j);
            }
            __syncthreads();
        }

        // ------------------------------------------------------------ S2
        // Claims, winners and grants for destinations in rows -1 .. RT.
        for (int u = threadIdx.x; u < AROWS * SS; u += NT) {
            const int ai = u / SS, si = u - ai * SS;  // ai = rr + 1
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
            if (ones && ai >= 1 && ai <= RT) sm.dirty[ai - 1] = 1u;
            sm.K[0][ai][si] = win[1] | win[3] | win[5] | win[7];
            sm.K[1][ai][si] = win[2] | win[3] | win[6] | win[7];
            sm.K[2][ai][si] = win[4] | win[5] | win[6] | win[7];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (win[q]) grant(sm, ai - 1, si, q, win[q]);
            if (twos) enqueue(sm, u, twos, 1);
        }
        __syncthreads();
        if (const uint32_t nq = sm.qc[1] & 0xFFFFu) {
            const uint32_t ne = sm.qc[1] >> 16;
            for (uint32_t e = threadIdx.x; e < nq; e += NT) {
                int u, j;
                list_entry(sm, ne, e, u, j);
                const int ai = u / SS, si = u - ai * SS;
                set_winner(sm, ai, si, j, draw_winner(a, sm, ai, si, j, r0, c0, seed, step));
            }
            __syncthreads();
        }

        // ------------------------------------------------------------ S3
        for (int rr = warp; rr < RT; rr += NW) {
            const int lr = r0 + rr;
            if (lr >= a.rows_owned) break;
            const int b = kGhost + lr;
            const int grow = a.row_begin + lr;
            const int rs = slot(base, rr + 3), ai = rr + 1;
            if (!ACO && !sm.dirty[rr]) {
                // Nothing arrives or leaves in this row: copy its 256 words
                // with 16-byte shared loads / global stores (lane = 4 columns).
                // (Not for ACO: the extra live registers cost it more in spills.)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = 128 * h + 4 * lane;
                    if (c0 + col < W)  // W is a multiple of 16: a 4-word group is all in or all out
                        *reinterpret_cast<uint4*>(cout + size_t(b) * W + c0 + col) =
                            *reinterpret_cast<const uint4*>(&sm.word[rs][HALO + col]);
                }
                continue;
            }
            const size_t row0 = size_t(b) * W + c0 + lane;  // this lane's cell in segment 1
            // ACO: issue the whole row's pheromone loads before using any of them.
            double2 tv[NS];
            if (ACO) {
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    tv[s] = (c0 + 32 * s + lane < W) ? tin[row0 + 32 * s] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int si = 1; si <= NS; ++si) {
                const int gc = c0 + 32 * (si - 1) + lane;
                const bool valid = gc < W;
                const uint32_t Am = sm.A[ai][si], Gm = sm.G[rr][si];
                const uint32_t w = sm.word[rs][si * 32 + lane - WOFF];
                const size_t gi = row0 + 32 * (si - 1);
                if ((Am | Gm) == 0u) {  // warp-uniform: nothing moves in this segment
                    if (valid) {
                        cout[gi] = w;
                        if (ACO) {
                            const double2 tt = tv[si - 1];
                            tout[gi] = make_double2(__dmul_rn(tt.x, a.k.factor), __dmul_rn(tt.y, a.k.factor));
                        }
                    }
                    continue;
                }
                uint32_t nw = w;
                bool arrived = false;
                uint32_t group = 0;
                double tour_new = 0.0;
                if (bit(Am, lane)) {
                    const int kc = int(bit(sm.K[0][ai][si], lane) | bit(sm.K[1][ai][si], lane) << 1 |
                                       bit(sm.K[2][ai][si], lane) << 2);
                    const uint32_t sw = sm.word[slot(base, rr + 3 + kDR[kc])][si * 32 + lane + kDC[kc] - WOFF];
                    group = sw >> 30;
                    nw = sw;
                    if (!(sw & kCrossedBit) && crossed_at(group, grow, a.k.H, band)) {  // src/engine.cpp:163-170
                        nw |= kCrossedBit;
                        if (valid) {
                            if (group == 1u) ++ntop;
                            else ++nbot;
                        }
                    }
                    arrived = true;
                    if (valid) ++moved;
                    if (ACO && valid) {  // tour += 1 or sqrt(2) (src/engine.cpp:159-160)
                        const size_t si_src = size_t(b + kDR[kc]) * W + (gc + kDC[kc]);
                        tour_new = __dadd_rn(tour[si_src], is_diag(kc) ? a.k.diag : 1.0);
                        tour[gi] = tour_new;
                    }
                } else if (bit(Gm, lane)) {
                    nw = 0u;
                }
                if (valid) {
                    cout[gi] = nw;
                    if (ACO) {  // evaporate, then deposit (src/engine.cpp:124-131, src/aco.cpp:119-123)
                        double2 tt = tv[si - 1];
                        tt.x = __dmul_rn(tt.x, a.k.factor);
                        tt.y = __dmul_rn(tt.y, a.k.factor);
                        if (arrived) {
                            const double dep = __ddiv_rn(a.k.q, tour_new);
                            if (group == 1u) tt.x = __dadd_rn(tt.x, dep);
                            else tt.y = __dadd_rn(tt.y, dep);
                        }
                        tout[gi] = tt;
                    }
                }
            }
        }
        __syncthreads();  // end of tile: the window's slots may be refilled
        base = slot(base, RT);
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
    }
    item = sm.item;  // claimed during the last tile (visible after its barriers)
    if (!kCrossPrefetch && item < n_items) {
        // Small ring: the next item's window is loaded only now, into the
        // slots the finished item released.
        if (warp == 0) {
            const Item nit = decode_item(item, strips, n_chunks, n_tiles, a.tiles_per_cta, W);
            load_rows(sm, a, parity, nit, nit.t_first * RT, 0, 0, SR, &sm.mbar[nload & 1]);
        }
        __syncthreads();  // wall rows written by warp 0 are visible to all
    }
    if (item < n_items) ++nload;
    }  // work items
}

// Three CTAs per SM must fit the 196 KB shared-memory carve-out step (1 KB
// reserved per CTA): the next step up (228 KB) leaves 28 KB of L1 instead of
// 60 KB, and the ACO pheromone stream then loses ~15% (measured).
static_assert(sizeof(Smem) <= (196 * 1024) / 3 - 1024 - 64, "shared memory would cost 3 CTAs/SM their L1");

int configure_step_bits() {
    const int bytes = int(sizeof(Smem));
    if (cudaFuncSetAttribute(step_bits_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(step_bits_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
        return 1;
    return 0;
}

// Persistent grid: one CTA per (SM x 3) slot at most. Work items are chunks of
// up to 16 consecutive RT-row tiles of one strip of one replica, sized so
// there are about 4 items per CTA for load balance.
int launch_step_bits(const StepArgs& a, int slot_idx, int parity, cudaStream_t s) {
    const int strips = (a.k.W + NS * 32 - 1) / (NS * 32);
    const int n_tiles = (a.rows_owned + RT - 1) / RT;
    const long long ctas_max = (long long)a.num_sms * 3;
    const long long tiles = (long long)strips * n_tiles * a.replicas;
    StepArgs b = a;
    b.tiles_per_cta = int(std::max<long long>(1, std::min<long long>(16, tiles / (ctas_max * a.items_per_cta))));
    const long long items = (long long)strips * ((n_tiles + b.tiles_per_cta - 1) / b.tiles_per_cta) * a.replicas;
    dim3 grid(unsigned(std::min(items, ctas_max)));
    const size_t bytes = sizeof(Smem);
    if (a.k.model == 1) step_bits_kernel<true><<<grid, NT, bytes, s>>>(b, slot_idx, parity);
    else step_bits_kernel<false><<<grid, NT, bytes, s>>>(b, slot_idx, parity);
    return 1;
}

}  // namespace pfk
