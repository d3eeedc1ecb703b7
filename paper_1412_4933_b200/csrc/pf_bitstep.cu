// Bit-sliced fused step kernel (the default product path, PF_KERNEL_FUSED).
//
// One CTA owns RT rows x NS 32-column segments of the grid. The per-step
// update (StepEngine::step, src/engine.cpp:53-193) is evaluated on 32-cell
// row segments held as 32-bit masks, so the common work costs one ALU op per
// 32 cells; only agents that must draw (forward blocked, some slot open) and
// destinations with >= 2 claimants fall to per-cell scalar code, and those are
// compacted into shared-memory work lists so every lane of the CTA takes one.
//
//   S0 stage   warp per segment-row, lane = column: load the step-start cell
//              words (3-row / 1-segment halo) into shared memory and ballot
//              them into occupancy planes v30 / v31 (bits 30/31 of the word:
//              Top = v30 & ~v31, Bottom = v31 & ~v30, Empty = ~(v30 | v31)).
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
#include "pf_internal.h"

namespace pfk {

using namespace pfdev;

namespace {

constexpr int RT = 32;           // output rows per CTA
constexpr int NS = 8;            // output 32-column segments per CTA
constexpr int SR = RT + 6;       // staged rows: -3 .. RT+2
constexpr int SS = NS + 2;       // staged segments: -1 .. NS
constexpr int SW = SS * 32;      // staged columns
constexpr int NT = 256;          // threads per CTA
constexpr int NW = NT / 32;
constexpr int DROWS = RT + 4;    // intent rows -2 .. RT+1
constexpr int AROWS = RT + 2;    // resolution rows -1 .. RT
#ifndef PF_BITS_QCAP
#define PF_BITS_QCAP 1024
#endif
constexpr int QCAP = PF_BITS_QCAP;  // work-list capacity (overflow is handled in place)

struct Smem {
    uint32_t word[SR][SW];  // rows are 1,280 B: every row start is 16-byte aligned for TMA
    unsigned long long mbar;
    uint32_t v30[SR][SS];
    uint32_t v31[SR][SS];
    uint32_t D[8][DROWS][SS];
    uint32_t A[AROWS][SS];
    uint32_t K[3][AROWS][SS];
    uint32_t G[RT][SS];
    uint32_t queue[QCAP];  // (unit << 5) | bit
    uint32_t nq;
    uint32_t cnt[3];
};

__device__ __forceinline__ uint32_t bit(uint32_t x, int j) { return (x >> j) & 1u; }

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

// Value of a plane at column c-1 (shift in from the left segment) / c+1.
__device__ __forceinline__ uint32_t from_left(uint32_t x, uint32_t left) { return (x << 1) | (left >> 31); }
__device__ __forceinline__ uint32_t from_right(uint32_t x, uint32_t right) { return (x >> 1) | (right << 31); }

// Emptiness around one intent unit (row di-2, segment si): the eight
// neighbour planes, shifted so bit j is the neighbour of column j.
struct Around {
    uint32_t em, emL, emR, e0L, e0R, ep, epL, epR;
};

__device__ __forceinline__ Around around(const Smem& sm, int sr, int si) {
    auto E = [&](int row, int seg) -> uint32_t {
        return (seg < 0 || seg >= SS) ? 0u : ~(sm.v30[row][seg] | sm.v31[row][seg]);
    };
    Around n;
    n.em = E(sr - 1, si);
    n.ep = E(sr + 1, si);
    const uint32_t e0 = E(sr, si);
    n.emL = from_left(n.em, E(sr - 1, si - 1));
    n.emR = from_right(n.em, E(sr - 1, si + 1));
    n.e0L = from_left(e0, E(sr, si - 1));
    n.e0R = from_right(e0, E(sr, si + 1));
    n.epL = from_left(n.ep, E(sr + 1, si - 1));
    n.epR = from_right(n.ep, E(sr + 1, si + 1));
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

// Append the set bits of `mask` for unit u to the work list; returns the bits
// that did not fit (to be processed in place).
__device__ __forceinline__ uint32_t enqueue(Smem& sm, int u, uint32_t mask) {
    const uint32_t n = __popc(mask);
    const uint32_t pos = atomicAdd(&sm.nq, n);
    uint32_t overflow = 0u;
    for (uint32_t i = 0; i < n; ++i) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1u;
        if (pos + i < uint32_t(QCAP)) sm.queue[pos + i] = (uint32_t(u) << 5) | uint32_t(j);
        else overflow |= 1u << j;
    }
    return overflow;
}

}  // namespace

// Intent of the draw-path agent at bit j of intent unit (di, si):
// lem_select / aco_select (src/lem.cpp:28-60, src/aco.cpp:64-92).
template <bool ACO>
__device__ __forceinline__ int draw_intent(const StepArgs& a, const Smem& sm, const double2* __restrict__ tin, int di,
                                           int si, int j, bool bottom, int r0, int c0, uint64_t seed, uint32_t step) {
    const int sr = di + 1;
    const Around n = around(sm, sr, si);
    uint32_t open;  // goal-relative slots F FL FR L R B BL BR
    if (!bottom)
        open = bit(n.ep, j) | bit(n.epL, j) << 1 | bit(n.epR, j) << 2 | bit(n.e0L, j) << 3 | bit(n.e0R, j) << 4 |
               bit(n.em, j) << 5 | bit(n.emL, j) << 6 | bit(n.emR, j) << 7;
    else
        open = bit(n.em, j) | bit(n.emR, j) << 1 | bit(n.emL, j) << 2 | bit(n.e0R, j) << 3 | bit(n.e0L, j) << 4 |
               bit(n.ep, j) << 5 | bit(n.epR, j) << 6 | bit(n.epL, j) << 7;
    const uint32_t id = sm.word[sr][si * 32 + j] & kIdMask;
    int s;
    if (!ACO) {
        s = lem_choose(a.kc, open, seed, step, id);
    } else {
        const int W = a.k.W;
        const int b = kGhost + r0 + di - 2;
        const int c = c0 + 32 * (si - 1) + j;
        double num[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            num[i] = 0.0;
            if (open >> i & 1u) {
                const uint8_t code = bottom ? uint8_t(7 - kSlotCodeTop[i]) : kSlotCodeTop[i];
                const double* t = reinterpret_cast<const double*>(tin + size_t(b + kDR[code]) * W + (c + kDC[code]));
                num[i] = __dmul_rn(pheromone_term(a.kc, __ldg(t + (bottom ? 1 : 0))), __ldg(&a.kc->eta[i]));
            }
        }
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

template <bool ACO>
__global__ void __launch_bounds__(NT, 3) step_bits_kernel(const StepArgs a, int slot, int parity) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    const int W = a.k.W;
    const int rep = blockIdx.z;
    const int r0 = blockIdx.y * RT;         // owned-local row of the tile
    const int c0 = blockIdx.x * (NS * 32);  // first owned column
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t step = *a.d_step + uint32_t(slot);
    const uint64_t seed = a.seed_base + uint64_t(rep);
    const size_t base = size_t(rep) * a.p.plane;
    const uint32_t* __restrict__ cin = a.p.cell[parity] + base;
    uint32_t* __restrict__ cout = a.p.cell[parity ^ 1] + base;
    const double2* __restrict__ tin = ACO ? a.p.tau[parity] + base : nullptr;
    double2* __restrict__ tout = ACO ? a.p.tau[parity ^ 1] + base : nullptr;
    double* __restrict__ tour = ACO ? a.p.tour + base : nullptr;

    // ---------------------------------------------------------------- S0
    // The staged rows arrive by TMA bulk copies (one cp.async.bulk per row,
    // completion counted on one mbarrier); columns / rows outside the arena
    // are filled with walls by the threads meanwhile.
    const int col_lo = max(c0 - 32, 0), col_hi = min(c0 + 32 * (NS + 1), W);  // multiples of 16
    const int fill_lo = col_lo - (c0 - 32), fill_hi = col_hi - (c0 - 32);      // staged column range
    const int rows_valid = max(0, min(SR, a.rows_buf - (kGhost + r0 - 3)));
    if (threadIdx.x == 0) {
        mbar_init(&sm.mbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) mbar_expect_tx(&sm.mbar, uint32_t(rows_valid) * uint32_t(fill_hi - fill_lo) * 4u);
        __syncwarp();
        for (int sr = lane; sr < rows_valid; sr += 32) {
            const int b = kGhost + r0 - 3 + sr;
            bulk_g2s(&sm.word[sr][fill_lo], cin + size_t(b) * W + col_lo, uint32_t(fill_hi - fill_lo) * 4u, &sm.mbar);
        }
    }
    for (int i = threadIdx.x; i < RT * SS; i += NT) (&sm.G[0][0])[i] = 0u;
    if (threadIdx.x < 3) sm.cnt[threadIdx.x] = 0u;
    if (threadIdx.x == 0) sm.nq = 0u;
    if (fill_lo > 0 || fill_hi < SW)
        for (int sr = warp; sr < rows_valid; sr += NW)
            for (int c = lane; c < SW; c += 32)
                if (c < fill_lo || c >= fill_hi) sm.word[sr][c] = kWall;
    for (int i = rows_valid * SW + threadIdx.x; i < SR * SW; i += NT) (&sm.word[0][0])[i] = kWall;
    mbar_wait(&sm.mbar, 0);
    __syncthreads();
    for (int sr = warp; sr < SR; sr += NW) {
        uint32_t m30 = 0u, m31 = 0u;  // lane si keeps segment si's planes
#pragma unroll
        for (int si = 0; si < SS; ++si) {
            const uint32_t w = sm.word[sr][si * 32 + lane];
            const uint32_t b30 = __ballot_sync(0xFFFFFFFFu, int32_t(w << 1) < 0);
            const uint32_t b31 = __ballot_sync(0xFFFFFFFFu, int32_t(w) < 0);
            m30 = lane == si ? b30 : m30;
            m31 = lane == si ? b31 : m31;
        }
        if (lane < SS) {
            sm.v30[sr][lane] = m30;
            sm.v31[sr][lane] = m31;
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- S1
    // Intents for rows -2 .. RT+1, all staged segments (halo segments only
    // at the two columns next to the tile).
    for (int u = threadIdx.x; u < DROWS * SS; u += NT) {
        const int di = u / SS, si = u - di * SS;  // di = rr + 2
        const int sr = di + 1;                    // staged row of rr
        const Around n = around(sm, sr, si);
        const uint32_t v30 = sm.v30[sr][si], v31 = sm.v31[sr][si];
        const uint32_t segmask = si == 0 ? 0xC0000000u : (si == SS - 1 ? 0x00000003u : 0xFFFFFFFFu);
        const uint32_t T = v30 & ~v31 & segmask, B = v31 & ~v30 & segmask;
        uint32_t d[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) d[k] = 0u;
        d[6] = T & n.ep;  // Top forward: (+1, 0)
        d[1] = B & n.em;  // Bottom forward: (-1, 0)
        const uint32_t any8 = n.ep | n.epL | n.epR | n.e0L | n.e0R | n.em | n.emL | n.emR;
        uint32_t slow = ((T & ~n.ep) | (B & ~n.em)) & any8;
        if (slow) slow = enqueue(sm, u, slow);
        while (slow) {  // queue overflow: draw in place
            const int j = __ffs(slow) - 1;
            slow &= slow - 1u;
            d[draw_intent<ACO>(a, sm, tin, di, si, j, bit(B, j) != 0u, r0, c0, seed, step)] |= 1u << j;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) sm.D[k][di][si] = d[k];
    }
    __syncthreads();
    {
        const uint32_t nq = min(sm.nq, uint32_t(QCAP));
        for (uint32_t e = threadIdx.x; e < nq; e += NT) {
            const uint32_t q = sm.queue[e];
            const int u = int(q >> 5), j = int(q & 31u);
            const int di = u / SS, si = u - di * SS;
            const bool bottom = bit(sm.v31[di + 1][si], j) != 0u;
            const int code = draw_intent<ACO>(a, sm, tin, di, si, j, bottom, r0, c0, seed, step);
            atomicOr(&sm.D[code][di][si], 1u << j);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sm.nq = 0u;
    __syncthreads();

    // ---------------------------------------------------------------- S2
    // Claims, winners and grants for destinations in rows -1 .. RT.
    for (int u = threadIdx.x; u < AROWS * SS; u += NT) {
        const int ai = u / SS, si = u - ai * SS;  // ai = rr + 1
        uint32_t C[8];
        claims(sm, ai, si, C);
        uint32_t ones = 0u, twos = 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            twos |= ones & C[k];
            ones |= C[k];
        }
        uint32_t win[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) win[k] = C[k] & ~twos;
        sm.A[ai][si] = ones;
        sm.K[0][ai][si] = win[1] | win[3] | win[5] | win[7];
        sm.K[1][ai][si] = win[2] | win[3] | win[6] | win[7];
        sm.K[2][ai][si] = win[4] | win[5] | win[6] | win[7];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (win[k]) grant(sm, ai - 1, si, k, win[k]);
        uint32_t multi = twos ? enqueue(sm, u, twos) : 0u;
        while (multi) {  // queue overflow: draw in place
            const int j = __ffs(multi) - 1;
            multi &= multi - 1u;
            set_winner(sm, ai, si, j, draw_winner(a, sm, ai, si, j, r0, c0, seed, step));
        }
    }
    __syncthreads();
    {
        const uint32_t nq = min(sm.nq, uint32_t(QCAP));
        for (uint32_t e = threadIdx.x; e < nq; e += NT) {
            const uint32_t q = sm.queue[e];
            const int u = int(q >> 5), j = int(q & 31u);
            const int ai = u / SS, si = u - ai * SS;
            set_winner(sm, ai, si, j, draw_winner(a, sm, ai, si, j, r0, c0, seed, step));
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- S3
    uint32_t moved = 0, ntop = 0, nbot = 0;
    for (int rr = warp; rr < RT; rr += NW) {
        const int lr = r0 + rr;
        if (lr >= a.rows_owned) break;
        const int b = kGhost + lr;
        const int grow = a.row_begin + lr;
        const int sr = rr + 3, ai = rr + 1;
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
            const uint32_t w = sm.word[sr][si * 32 + lane];
            const size_t gi = row0 + 32 * (si - 1);
            if ((Am | Gm) == 0u) {  // warp-uniform: nothing moves in this segment
                if (valid) {
                    cout[gi] = w;
                    if (ACO) {
                        const double2 t = tv[si - 1];
                        tout[gi] = make_double2(__dmul_rn(t.x, a.k.factor), __dmul_rn(t.y, a.k.factor));
                    }
                }
                continue;
            }
            uint32_t nw = w;
            bool arrived = false;
            uint32_t group = 0;
            double tour_new = 0.0;
            if (bit(Am, lane)) {
                const int k = int(bit(sm.K[0][ai][si], lane) | bit(sm.K[1][ai][si], lane) << 1 |
                                  bit(sm.K[2][ai][si], lane) << 2);
                const uint32_t sw = sm.word[sr + kDR[k]][si * 32 + lane + kDC[k]];
                group = sw >> 30;
                nw = sw;
                if (!(sw & kCrossedBit) && crossed_at(group, grow, a.k.H, a.k.band)) {
                    nw |= kCrossedBit;
                    if (valid) {
                        if (group == 1u) ++ntop;
                        else ++nbot;
                    }
                }
                arrived = true;
                if (valid) ++moved;
                if (ACO && valid) {
                    const size_t si_src = size_t(b + kDR[k]) * W + (gc + kDC[k]);
                    tour_new = __dadd_rn(tour[si_src], is_diag(k) ? a.k.diag : 1.0);
                    tour[gi] = tour_new;
                }
            } else if (bit(Gm, lane)) {
                nw = 0u;
            }
            if (valid) {
                cout[gi] = nw;
                if (ACO) {
                    double2 t = tv[si - 1];
                    t.x = __dmul_rn(t.x, a.k.factor);
                    t.y = __dmul_rn(t.y, a.k.factor);
                    if (arrived) {
                        const double dep = __ddiv_rn(a.k.q, tour_new);
                        if (group == 1u) t.x = __dadd_rn(t.x, dep);
                        else t.y = __dadd_rn(t.y, dep);
                    }
                    tout[gi] = t;
                }
            }
        }
    }
    moved = __reduce_add_sync(0xFFFFFFFFu, moved);
    ntop = __reduce_add_sync(0xFFFFFFFFu, ntop);
    nbot = __reduce_add_sync(0xFFFFFFFFu, nbot);
    if (lane == 0 && (moved | ntop | nbot)) {
        atomicAdd(&sm.cnt[0], moved);
        atomicAdd(&sm.cnt[1], ntop);
        atomicAdd(&sm.cnt[2], nbot);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* rep_slot = a.reports + (size_t(rep) * a.report_cap + step % uint32_t(a.report_cap)) * 4;
        if (blockIdx.x == 0 && blockIdx.y == 0) rep_slot[0] = step;
        if (sm.cnt[0]) atomicAdd(&rep_slot[1], sm.cnt[0]);
        if (sm.cnt[1]) atomicAdd(&rep_slot[2], sm.cnt[1]);
        if (sm.cnt[2]) atomicAdd(&rep_slot[3], sm.cnt[2]);
    }
}

int configure_step_bits() {
    const int bytes = int(sizeof(Smem));
    if (cudaFuncSetAttribute(step_bits_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(step_bits_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
        return 1;
    return 0;
}

int launch_step_bits(const StepArgs& a, int slot, int parity, cudaStream_t s) {
    dim3 grid((a.k.W + NS * 32 - 1) / (NS * 32), (a.rows_owned + RT - 1) / RT, a.replicas);
    const size_t bytes = sizeof(Smem);
    if (a.k.model == 1) step_bits_kernel<true><<<grid, NT, bytes, s>>>(a, slot, parity);
    else step_bits_kernel<false><<<grid, NT, bytes, s>>>(a, slot, parity);
    return 1;
}

}  // namespace pfk
