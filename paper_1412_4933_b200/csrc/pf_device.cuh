// Device-side building blocks of the per-step update: the keyed Philox
// stream, the AS241 quantile, and the per-agent move proposal (LEM / ACO).
//
// Every floating-point operation uses an explicit round-to-nearest intrinsic
// (__dmul_rn, __dadd_rn, ...) in the reference's evaluation order, so no FMA
// contraction can change a bit; the library is additionally built with
// --fmad=false. The AS241 tail's log is glibc's algorithm restated
// (glibc_log); the only non-IEEE-exact call left is pow() for ACO alpha not
// in {0, 1}; see DESIGN.md "Bit-exactness".
#pragma once

#include <cstdint>

#include <math_constants.h>

#include "pf_glibc_log.h"

namespace pfdev {

// Cell word: agent id in bits 0..28, crossed flag bit 29, group in bits 30..31
// (1 = Top, 2 = Bottom). 0 = empty; kWall (group 3) = outside the arena.
constexpr uint32_t kIdMask = 0x1FFFFFFFu;
constexpr uint32_t kCrossedBit = 1u << 29;
constexpr uint32_t kWall = 0xFFFFFFFFu;
constexpr uint8_t kNone = 0xFF;

enum : uint32_t { kPhasePlacement = 0, kPhaseLemSelect = 1, kPhaseAcoSelect = 2, kPhaseResolve = 3, kPhaseTieBreak = 4 };

// Row-major neighbour codes around a cell (the reference's contender scan
// order, src/engine.cpp:15-24): code j <-> offset (kDR[j], kDC[j]); the
// opposite direction of code j is 7 - j.
static __device__ __constant__ const int8_t kDR[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static __device__ __constant__ const int8_t kDC[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

// Goal-relative slot i (F FL FR L R B BL BR, inc/grid.hpp:19-43) -> row-major
// code, for a Top agent. A Bottom agent's slot is the point reflection
// (inc/grid.hpp:45-49), whose code is 7 - the Top code.
static __device__ __constant__ const uint8_t kSlotCodeTop[8] = {6, 5, 7, 3, 4, 1, 0, 2};

struct StepConsts {
    double lem_score[8]; // d_min / d_i (src/lem.cpp:8-18), host-computed
    double eta[8];       // (1/d_i)^beta (src/aco.cpp:20-27), host-computed
    double sel_mu, sel_sigma;
    double alpha;
    int alpha_mode;      // 0: tau, 1: 1.0, 2: pow(tau, alpha) (src/aco.cpp:31-35)
    double factor;       // 1 - rho (src/engine.cpp:126)
    double q;
    double diag;         // sqrt(2) (src/aco.cpp:11)
    int model;           // 0 LEM, 1 ACO
    int W, H;
};

// Per-replica scenario parameters: replicas of one context share the grid and
// the model but may differ in seed and density (sweep, tools/pedflow.cpp:159-189).
struct ReplicaParams {
    uint64_t seed;      // RngKey seed (inc/rng.hpp:9-37)
    int32_t band;       // band_height(agents_per_side, W) (src/metrics.cpp:8-11)
    uint32_t n_agents;  // 2 * agents_per_side
};

// ----------------------------------------------------------------- Philox

// Philox4x32-10 with the reference's packing (src/rng.cpp:43-55).
__device__ __forceinline__ uint64_t philox_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity,
                                                uint32_t counter) {
    uint32_t c0 = uint32_t(entity), c1 = uint32_t(entity >> 32), c2 = step;
    uint32_t c3 = (phase << 28) | (counter & 0x0FFFFFFFu);
    uint32_t k0 = uint32_t(seed), k1 = uint32_t(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c1 = lo1;
        c3 = lo0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return (uint64_t(c0) << 32) | c1;
}

// uniform(): (bits >> 11) * 2^-53 (src/rng.cpp:57-59). Exact.
__device__ __forceinline__ double uniform_from_bits(uint64_t bits) {
    return __dmul_rn(__ull2double_rn(bits >> 11), 0x1.0p-53);
}

__device__ __forceinline__ double horner8(const double (&c)[8], double r) {
    double v = c[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) v = __dadd_rn(__dmul_rn(v, r), c[i]);
    return v;
}

// glibc's log (the reference's std::log, src/rng.cpp:93-96) restated op for
// op: the main path of sysdeps/ieee754/dbl-64/e_log.c (N = 128 table) in the
// order and with the FMA contractions of the -mfma build (__log_fma) that
// this image's glibc 2.39 dispatches to on FMA + AVX2 hosts, constants from
// its libm (pf_glibc_log.h, tools/gen_log_table.py). Bit-identical to the
// host's log for positive normal x away from 1 (checked on the host against
// libm by the oracle's pfo_log_restated, and device against host by
// tests/test_gpu_parity.py); the AS241 tail only asks for x in (0, 0.075].
// Outside that domain it falls back to CUDA's log (<= 1 ulp).
static __device__ const double kLogTab[128][2] = PF_LOG_TAB_INIT;
static __device__ const double kLogPoly[5] = PF_LOG_POLY_INIT;

// lt.tab(i, j) / lt.poly(i): kLogTab / kLogPoly (global memory, or a copy).
struct GlobalLogTab {
    __device__ double tab(int i, int j) const { return __ldg(&kLogTab[i][j]); }
    __device__ double poly(int i) const { return __ldg(&kLogPoly[i]); }
};

template <class LT>
__device__ __forceinline__ double glibc_log_with(const LT& lt, double x) {
    const uint64_t ix = uint64_t(__double_as_longlong(x));
    const uint64_t top = ix >> 48;
    if (ix - 0x3fee000000000000ull < 0x3ff1090000000000ull - 0x3fee000000000000ull || top - 0x0010u >= 0x7ff0u - 0x0010u)
        return log(x);
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = int((tmp >> 45) & 127u);
    const int k = int(int64_t(tmp) >> 52);
    const double z = __longlong_as_double((long long)(ix - (tmp & (0xfffull << 52))));
    const double kd = double(k);
    const double w = __fma_rn(kd, PF_LOG_LN2HI, lt.tab(i, 1));
    const double r = __fma_rn(z, lt.tab(i, 0), -1.0);
    const double p21 = __fma_rn(r, lt.poly(2), lt.poly(1));
    const double hi = __dadd_rn(r, w);
    const double r2 = __dmul_rn(r, r);
    double lo = __dadd_rn(__dsub_rn(w, hi), r);
    lo = __fma_rn(kd, PF_LOG_LN2LO, lo);
    const double r3 = __dmul_rn(r, r2);
    double p43 = __fma_rn(r, lt.poly(4), lt.poly(3));
    lo = __fma_rn(r2, lt.poly(0), lo);
    p43 = __fma_rn(p43, r2, p21);
    return __dadd_rn(__fma_rn(r3, p43, lo), hi);
}

__device__ __forceinline__ double glibc_log(double x) { return glibc_log_with(GlobalLogTab{}, x); }

// Wichura AS241 PPND16 (src/rng.cpp:61-150), same coefficients and order.
template <class LT>
__device__ __forceinline__ double inverse_normal_cdf_with(const LT& lt, double p) {
    const double q = __dsub_rn(p, 0.5);
    if (fabs(q) <= 0.425) {
        constexpr double num[8] = {2.5090809287301226727e3, 3.3430575583588128105e4, 6.7265770927008700853e4,
                                   4.5921953931549871457e4, 1.3731693765509461125e4, 1.9715909503065514427e3,
                                   1.3314166789178437745e2, 3.3871328727963666080e0};
        constexpr double den[8] = {5.2264952788528545610e3, 2.8729085735721942674e4, 3.9307895800092710610e4,
                                   2.1213794301586595867e4, 5.3941960214247511077e3, 6.8718700749205790830e2,
                                   4.2313330701600911252e1, 1.0};
        const double r = __dsub_rn(0.180625, __dmul_rn(q, q));
        return __ddiv_rn(__dmul_rn(q, horner8(num, r)), horner8(den, r));
    }
    double r = (q < 0.0) ? p : __dsub_rn(1.0, p);
    r = __dsqrt_rn(-glibc_log_with(lt, r));
    double val;
    if (r <= 5.0) {
        constexpr double num[8] = {7.74545014278341407640e-4, 2.27238449892691845833e-2, 2.41780725177450611770e-1,
                                   1.27045825245236838258e0,  3.64784832476320460504e0,  5.76949722146069140550e0,
                                   4.63033784615654529590e0,  1.42343711074968357734e0};
        constexpr double den[8] = {1.05075007164441684324e-9, 5.47593808499534494600e-4, 1.51986665636164571966e-2,
                                   1.48103976427480074590e-1, 6.89767334985100004550e-1, 1.67638483018380384940e0,
                                   2.05319162663775882187e0,  1.0};
        r = __dsub_rn(r, 1.6);
        val = __ddiv_rn(horner8(num, r), horner8(den, r));
    } else {
        constexpr double num[8] = {2.01033439929228813265e-7, 2.71155556874348757815e-5, 1.24266094738807843860e-3,
                                   2.65321895265761230930e-2, 2.96560571828504891230e-1, 1.78482653991729133580e0,
                                   5.46378491116411436990e0,  6.65790464350110377720e0};
        constexpr double den[8] = {2.04426310338993978564e-15, 1.42151175831644588870e-7, 1.84631831751005468180e-5,
                                   7.86869131145613259100e-4,  1.48753612908506148525e-2, 1.36929880922735805310e-1,
                                   5.99832206555887937690e-1,  1.0};
        r = __dsub_rn(r, 5.0);
        val = __ddiv_rn(horner8(num, r), horner8(den, r));
    }
    return (q < 0.0) ? -val : val;
}

static __device__ __noinline__ double inverse_normal_cdf(double p) { return inverse_normal_cdf_with(GlobalLogTab{}, p); }


// ----------------------------------------------------------- proposals

// Slow path of lem_select (src/lem.cpp:28-60): the forward slot is blocked
// and at least one slot is open. Returns the chosen goal-relative slot.
// Inlined into the draw loops (A/B: C4 x64 -9%, C5 LEM -6%); the rarely
// divergent AS241 tail stays out of line.
// tab.score(i), tab.mu(), tab.sigma() return lem_score[i], sel_mu and
// sel_sigma (the step constants, from global memory or a shared-memory copy);
// tab.normal(u) is inverse_normal_cdf(u).
template <class Tab>
__device__ __forceinline__ int lem_choose_with(const Tab& tab, uint32_t open, uint64_t seed, uint32_t step,
                                               uint32_t id) {
    // C_max = the largest open score (src/lem.cpp:28-30). With d0 > 1
    // (validate) the distance table grows with the slot index (d_F < d_FL <
    // d_L < d_B < d_BL) and dmin/d_i shrinks, so that is the first open
    // slot's score (host-checked in fill_consts).
    const double cmax = tab.score(__ffs(open) - 1);
    // Tab::kEagerTie: the tie-break bits drawn up front, independent of (and
    // interleaved with) the selection draw, instead of after the gap scan.
    [[maybe_unused]] uint64_t tie_bits;
    if constexpr (Tab::kEagerTie) tie_bits = philox_bits(seed, step, kPhaseTieBreak, id, 0);
    // normal(key, mu_sel*C_max, sigma_sel*C_max) (src/lem.cpp:34, src/rng.cpp:152-156)
    const uint64_t bits = philox_bits(seed, step, kPhaseLemSelect, id, 0);
    const double u = __dmul_rn(__dadd_rn(__ull2double_rn(bits >> 11), 0.5), 0x1.0p-53);
    const double mu = __dmul_rn(tab.mu(), cmax), sg = __dmul_rn(tab.sigma(), cmax);
    double r = __dadd_rn(mu, __dmul_rn(sg, tab.normal(u)));
    r = (r < 0.0) ? 0.0 : ((cmax < r) ? cmax : r); // std::clamp(r, 0, C_max)
    // The open slot(s) nearest r (src/lem.cpp:38-52). The reference's scan
    // (reset on a strictly smaller gap, append on an equal one) ends with
    // exactly the open slots whose gap equals the minimum, in canonical
    // order; here that set is built branch-free as a bit mask.
    double gap[8];
    double best = CUDART_INF;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        gap[i] = (open >> i & 1u) ? fabs(__dsub_rn(tab.score(i), r)) : CUDART_INF;
        best = (gap[i] < best) ? gap[i] : best;
    }
    uint32_t tied = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) tied |= uint32_t((open >> i & 1u) != 0u && gap[i] == best) << i;
    const int ntied = __popc(tied);
    if (ntied > 1) {  // tie break: uniform(key.with_phase(TieBreak)) (src/lem.cpp:54-58)
        double tu;
        if constexpr (Tab::kEagerTie) tu = uniform_from_bits(tie_bits);
        else tu = uniform_from_bits(philox_bits(seed, step, kPhaseTieBreak, id, 0));
        int j = __double2int_rz(__dmul_rn(tu, double(ntied)));
        j = j < ntied - 1 ? j : ntied - 1;
        for (int t = 0; t < j; ++t) tied &= tied - 1u;  // drop the j lowest
    }
    return __ffs(tied) - 1;
}

// The step constants in global memory (read-only path).
struct GlobalLemTab {
    static constexpr bool kEagerTie = false;
    const StepConsts* k;
    __device__ double score(int i) const { return __ldg(&k->lem_score[i]); }
    __device__ double mu() const { return __ldg(&k->sel_mu); }
    __device__ double sigma() const { return __ldg(&k->sel_sigma); }
    __device__ double normal(double u) const { return inverse_normal_cdf(u); }
};

static __device__ __forceinline__ int lem_choose(const StepConsts* __restrict__ k, uint32_t open, uint64_t seed,
                                       uint32_t step, uint32_t id) {
    return lem_choose_with(GlobalLemTab{k}, open, seed, step, id);
}

// Slow path of aco_select (src/aco.cpp:64-92) given the numerators of the
// open slots (aco_numerators, src/aco.cpp:39-51).
static __device__ __forceinline__ int aco_choose(const double (&num)[8], uint32_t open, uint64_t seed, uint32_t step,
                                       uint32_t id) {
    // Closed slots count as exact zeros (aco_numerators gives them 0,
    // src/aco.cpp:39-51), and adding an exact zero changes no sum, so the
    // candidates' sequential sums (src/aco.cpp:65-72, 80-89) are the running
    // sums over all eight slots in canonical order. The first slot whose
    // running sum exceeds u * total is open (a closed slot adds nothing), so
    // the pick is the lowest set bit of a branch-free mask.
    double v[8];
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = (open >> i & 1u) ? num[i] : 0.0;
        total = __dadd_rn(total, v[i]);
    }
    const int k = __popc(open), last = 31 - __clz(open);
    const double u = uniform_from_bits(philox_bits(seed, step, kPhaseAcoSelect, id, 0));
    if (total <= 0.0) {  // src/aco.cpp:77-79
        int j = __double2int_rz(__dmul_rn(u, double(k)));
        j = j < k - 1 ? j : k - 1;
        uint32_t m = open;
        for (int t = 0; t < j; ++t) m &= m - 1u;
        return __ffs(m) - 1;
    }
    const double target = __dmul_rn(u, total);
    double cum = 0.0;
    uint32_t over = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        cum = __dadd_rn(cum, v[i]);
        over |= uint32_t(cum > target) << i;
    }
    return over ? __ffs(over) - 1 : last;
}

__device__ __forceinline__ double pheromone_term(const StepConsts* __restrict__ k, double tau) {
    const int mode = __ldg(&k->alpha_mode);
    if (mode == 0) return tau;
    if (mode == 1) return 1.0;
    return pow(tau, __ldg(&k->alpha)); // alpha not in {0,1}: tolerance-only parity
}

// Proposal of the agent with cell word `word` (score_phase + intention_phase,
// src/engine.cpp:64-90). cell_at(dr, dc) returns the step-start word of the
// neighbour (kWall outside the arena); tau_at(dr, dc, group) returns that
// neighbour's own-group pheromone. Returns the row-major code of the target
// cell, or kNone to stay.
template <class CellAt, class TauAt>
__device__ __forceinline__ uint8_t propose(const StepConsts* __restrict__ k, int model, uint32_t word, uint64_t seed, uint32_t step,
                                           CellAt cell_at, TauAt tau_at) {
    const uint32_t group = word >> 30;
    const bool bottom = group == 2u;
    // Forward priority: no draw (src/lem.cpp:23-26, src/aco.cpp:60-63).
    {
        const uint8_t cf = bottom ? uint8_t(7 - kSlotCodeTop[0]) : kSlotCodeTop[0];
        if (cell_at(kDR[cf], kDC[cf]) == 0u) return cf;
    }
    uint32_t open = 0;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        const uint8_t c = bottom ? uint8_t(7 - kSlotCodeTop[i]) : kSlotCodeTop[i];
        open |= uint32_t(cell_at(kDR[c], kDC[c]) == 0u) << i;
    }
    if (open == 0u) return kNone; // boxed in: stay
    const uint32_t id = word & kIdMask;
    int slot;
    if (model == 0) {
        slot = lem_choose(k, open, seed, step, id);
    } else {
        double num[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            num[i] = 0.0;
            if (open >> i & 1u) {
                const uint8_t c = bottom ? uint8_t(7 - kSlotCodeTop[i]) : kSlotCodeTop[i];
                num[i] = __dmul_rn(pheromone_term(k, tau_at(kDR[c], kDC[c], bottom)), __ldg(&k->eta[i]));
            }
        }
        slot = aco_choose(num, open, seed, step, id);
    }
    return bottom ? uint8_t(7 - kSlotCodeTop[slot]) : kSlotCodeTop[slot];
}

// Cell-centric conflict resolution for one destination whose claim mask has
// bit j set when the neighbour at row-major code j targets it (the gather of
// src/engine.cpp:101-122). Returns the code of the winning source.
__device__ __forceinline__ uint8_t resolve(uint32_t claims, uint64_t seed, uint32_t step, uint64_t gidx) {
    const int kc = __popc(claims);
    if (kc == 1) return uint8_t(__ffs(claims) - 1);
    const double u = uniform_from_bits(philox_bits(seed, step, kPhaseResolve, gidx, 0));
    int j = __double2int_rz(__dmul_rn(u, double(kc)));
    j = j < kc - 1 ? j : kc - 1;
    uint32_t m = claims;
    for (int t = 0; t < j; ++t) m &= m - 1u; // drop the j lowest contenders
    return uint8_t(__ffs(m) - 1);
}

// crossed() (src/metrics.cpp:13-16) for a mover landing on global row grow.
__device__ __forceinline__ bool crossed_at(uint32_t group, int grow, int H, int band) {
    return group == 1u ? grow >= H - band : grow <= band - 1;
}

__device__ __forceinline__ bool is_diag(int code) { return code == 0 || code == 2 || code == 5 || code == 7; }

} // namespace pfdev
