/* TEST INFRASTRUCTURE — NOT PRODUCT CODE. See pedflow_oracle.h.
 *
 * A sequential restatement of the reference's per-step update, written in
 * plain C from the reference's documented behaviour. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Built with -O2 -ffp-contract=off so every double operation rounds exactly
 * as the reference build does.
 */
#include "pedflow_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- det-rng */

/* Philox4x32-10 with the reference's key/counter packing (src/rng.cpp:12-55):
 * key = (seed lo, seed hi); ctr = (entity lo, entity hi, step,
 * phase<<28 | counter&0x0FFFFFFF); output = ctr0<<32 | ctr1. */
uint64_t pfo_random_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter) {
    uint32_t c0 = (uint32_t)entity, c1 = (uint32_t)(entity >> 32), c2 = step;
    uint32_t c3 = (phase << 28) | (counter & 0x0FFFFFFFu);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return ((uint64_t)c0 << 32) | c1;
}

/* src/rng.cpp:57-59 */
double pfo_uniform(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter) {
    return (double)(pfo_random_bits(seed, step, phase, entity, counter) >> 11) * 0x1.0p-53;
}

/* Wichura AS241 PPND16, src/rng.cpp:61-150: the same coefficients evaluated
 * in the same Horner order. */
static double horner8(const double* c, double r) {
    /* (((((((c0*r + c1)*r + c2)*r + c3)*r + c4)*r + c5)*r + c6)*r + c7 */
    double v = c[0];
    for (int i = 1; i < 8; ++i) v = v * r + c[i];
    return v;
}

static const double kCentralNum[8] = {2.5090809287301226727e3, 3.3430575583588128105e4,
                                      6.7265770927008700853e4, 4.5921953931549871457e4,
                                      1.3731693765509461125e4, 1.9715909503065514427e3,
                                      1.3314166789178437745e2, 3.3871328727963666080e0};
static const double kCentralDen[8] = {5.2264952788528545610e3, 2.8729085735721942674e4,
                                      3.9307895800092710610e4, 2.1213794301586595867e4,
                                      5.3941960214247511077e3, 6.8718700749205790830e2,
                                      4.2313330701600911252e1, 1.0};
static const double kNearNum[8] = {7.74545014278341407640e-4, 2.27238449892691845833e-2,
                                   2.41780725177450611770e-1, 1.27045825245236838258e0,
                                   3.64784832476320460504e0, 5.76949722146069140550e0,
                                   4.63033784615654529590e0, 1.42343711074968357734e0};
static const double kNearDen[8] = {1.05075007164441684324e-9, 5.47593808499534494600e-4,
                                   1.51986665636164571966e-2, 1.48103976427480074590e-1,
                                   6.89767334985100004550e-1, 1.67638483018380384940e0,
                                   2.05319162663775882187e0, 1.0};
static const double kFarNum[8] = {2.01033439929228813265e-7, 2.71155556874348757815e-5,
                                  1.24266094738807843860e-3, 2.65321895265761230930e-2,
                                  2.96560571828504891230e-1, 1.78482653991729133580e0,
                                  5.46378491116411436990e0, 6.65790464350110377720e0};
static const double kFarDen[8] = {2.04426310338993978564e-15, 1.42151175831644588870e-7,
                                  1.84631831751005468180e-5, 7.86869131145613259100e-4,
                                  1.48753612908506148525e-2, 1.36929880922735805310e-1,
                                  5.99832206555887937690e-1, 1.0};

/* glibc's log, main path (sysdeps/ieee754/dbl-64/e_log.c, N = 128), in the
 * order and with the FMA contractions of the -mfma build this image's libm
 * dispatches to on FMA + AVX2 hosts (__log_fma, glibc 2.39). Constants:
 * pf_glibc_log.h (tools/gen_log_table.py). */
#include "pf_glibc_log.h"
static const double kLogPoly[5] = PF_LOG_POLY_INIT;
static const double kLogTab[128][2] = PF_LOG_TAB_INIT;

double pfo_log_restated(double x) {
    uint64_t ix;
    memcpy(&ix, &x, 8);
    const uint64_t top = ix >> 48;
    if (ix - 0x3fee000000000000ULL < 0x3ff1090000000000ULL - 0x3fee000000000000ULL || top - 0x0010 >= 0x7ff0 - 0x0010)
        return NAN; /* near 1, or zero / subnormal / negative / inf / nan: not restated */
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;
    const int i = (int)((tmp >> 45) & 127);
    const int k = (int)((int64_t)tmp >> 52);
    const uint64_t iz = ix - (tmp & 0xfffULL << 52);
    double z;
    memcpy(&z, &iz, 8);
    const double kd = (double)k;
    const double w = fma(kd, PF_LOG_LN2HI, kLogTab[i][1]);
    const double r = fma(z, kLogTab[i][0], -1.0);
    const double p21 = fma(r, kLogPoly[2], kLogPoly[1]);
    const double hi = r + w;
    const double r2 = r * r;
    double lo = (w - hi) + r;
    lo = fma(kd, PF_LOG_LN2LO, lo);
    const double r3 = r * r2;
    double p43 = fma(r, kLogPoly[4], kLogPoly[3]);
    lo = fma(r2, kLogPoly[0], lo);
    p43 = fma(p43, r2, p21);
    const double y = fma(r3, p43, lo);
    return y + hi;
}

int pfo_log_restated_matches_host(uint32_t n, uint64_t seed) {
    for (uint32_t j = 0; j < n; ++j) {
        /* tail arguments of AS241: min(p, 1 - p) with p an open uniform, in (0, 0.075] */
        const double u = ((double)(pfo_random_bits(seed, j, 0, j, 0) >> 11) + 0.5) * 0x1.0p-53;
        const double x = u * 0.15 < 0.075 ? u * 0.15 : 0.075;
        const double a = pfo_log_restated(x), b = log(x);
        if (memcmp(&a, &b, 8) != 0) return 0;
    }
    return 1;
}

double pfo_inverse_normal_cdf(double p) {
    const double q = p - 0.5;
    if (fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        return q * horner8(kCentralNum, r) / horner8(kCentralDen, r);
    }
    double r = (q < 0.0) ? p : 1.0 - p;
    r = sqrt(-log(r));
    double val;
    if (r <= 5.0) {
        r -= 1.6;
        val = horner8(kNearNum, r) / horner8(kNearDen, r);
    } else {
        r -= 5.0;
        val = horner8(kFarNum, r) / horner8(kFarDen, r);
    }
    return (q < 0.0) ? -val : val;
}

/* src/rng.cpp:152-156: open-interval uniform then the quantile. */
double pfo_normal(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter,
                  double mu, double sigma) {
    const double u = ((double)(pfo_random_bits(seed, step, phase, entity, counter) >> 11) + 0.5) * 0x1.0p-53;
    return mu + sigma * pfo_inverse_normal_cdf(u);
}

void pfo_normal_batch(uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                      const uint64_t* entity, const uint32_t* counter, double mu, double sigma, double* out) {
    for (uint32_t i = 0; i < n; ++i) out[i] = pfo_normal(seed[i], step[i], phase[i], entity[i], counter[i], mu, sigma);
}

/* -------------------------------------------------------------- grid-core */

uint32_t pfo_agent_size(void) { return (uint32_t)sizeof(pfo_agent); }

/* Goal-relative offsets of a Top agent, slot order F FL FR L R B BL BR
 * (inc/grid.hpp:34-43); Bottom agents use the point reflection
 * (inc/grid.hpp:45-49). */
static const int kGoal[8][2] = {{+1, 0}, {+1, -1}, {+1, +1}, {0, -1}, {0, +1}, {-1, 0}, {-1, -1}, {-1, +1}};

/* Row-major neighbour scan order around a destination (src/engine.cpp:15-24). */
static const int kCellNb[8][2] = {{-1, -1}, {-1, 0}, {-1, +1}, {0, -1}, {0, +1}, {+1, -1}, {+1, 0}, {+1, +1}};

/* src/grid.cpp:10-27: d = sqrt((d0-f)^2 + l^2). */
int pfo_distance_table(double d0, double out[8]) {
    if (!(d0 > 1.0)) return 2;
    const int f[8] = {+1, +1, +1, 0, 0, -1, -1, -1};
    const int l[8] = {0, 1, 1, 1, 1, 0, 1, 1};
    for (int i = 0; i < 8; ++i) out[i] = sqrt((d0 - f[i]) * (d0 - f[i]) + (double)(l[i] * l[i]));
    return 0;
}

/* src/metrics.cpp:8-11 */
int32_t pfo_band_height(int32_t n, int32_t width) {
    if (width <= 0) return 0;
    return (int32_t)(((int64_t)n + width - 1) / width);
}

/* src/lem.cpp:8-18: dmin = d[F] regardless of occupancy. */
void pfo_lem_scores(const uint8_t open[8], const double d[8], double out[8]) {
    const double dmin = d[0];
    for (int i = 0; i < 8; ++i) out[i] = open[i] ? dmin / d[i] : 0.0;
}

/* src/aco.cpp:31-51 */
static double pheromone_term(double tau, double alpha) {
    if (alpha == 1.0) return tau;
    if (alpha == 0.0) return 1.0;
    return pow(tau, alpha);
}

void pfo_aco_numerators(const uint8_t open[8], const double tau[8], double alpha, const double eta[8],
                        double out[8]) {
    for (int i = 0; i < 8; ++i) out[i] = open[i] ? pheromone_term(tau[i], alpha) * eta[i] : 0.0;
}

/* src/lem.cpp:20-61, split into the draw and the deterministic choice so the
 * SPEC examples (SPEC.md lem_select) can be fed explicit draws. */
int pfo_lem_select_u(const double sc[8], const uint8_t open[8], double r, double tie_u) {
    if (open[0]) return 0;
    double cmax = 0.0;
    for (int i = 0; i < 8; ++i) cmax = (cmax < sc[i]) ? sc[i] : cmax; /* std::max */
    if (cmax <= 0.0) return -1;
    /* std::clamp(r, 0, cmax) */
    if (r < 0.0) r = 0.0;
    else if (cmax < r) r = cmax;
    double best = -1.0;
    int tied[8], ntied = 0;
    for (int i = 0; i < 8; ++i) {
        const double s = sc[i];
        if (s <= 0.0) continue;
        const double gap = fabs(s - r);
        if (ntied == 0 || gap < best) {
            best = gap;
            ntied = 0;
            tied[ntied++] = i;
        } else if (gap == best) {
            tied[ntied++] = i;
        }
    }
    if (ntied > 1) {
        int j = (int)(tie_u * ntied);
        if (j > ntied - 1) j = ntied - 1;
        return tied[j];
    }
    return tied[0];
}

int pfo_lem_select(const double sc[8], const uint8_t open[8], uint64_t seed, uint32_t step, uint64_t agent,
                   double mu_sel, double sigma_sel) {
    if (open[0]) return 0;
    double cmax = 0.0;
    for (int i = 0; i < 8; ++i) cmax = (cmax < sc[i]) ? sc[i] : cmax;
    if (cmax <= 0.0) return -1;
    const double r = pfo_normal(seed, step, PFO_LEM_SELECT, agent, 0, mu_sel * cmax, sigma_sel * cmax);
    /* The tie-break draw is only consumed when needed; evaluating it eagerly
     * is harmless because draws are pure functions of their key. */
    const double tie_u = pfo_uniform(seed, step, PFO_TIE_BREAK, agent, 0);
    return pfo_lem_select_u(sc, open, r, tie_u);
}

/* src/aco.cpp:59-93 */
int pfo_aco_select_u(const double sc[8], const uint8_t open[8], double u) {
    if (open[0]) return 0;
    int cand[8], k = 0;
    double total = 0.0;
    for (int i = 0; i < 8; ++i) {
        if (!open[i]) continue;
        cand[k++] = i;
        total += sc[i];
    }
    if (k == 0) return -1;
    int pick = cand[k - 1];
    if (total <= 0.0) {
        int j = (int)(u * k);
        if (j > k - 1) j = k - 1;
        pick = cand[j];
    } else {
        double cum = 0.0;
        for (int j = 0; j < k; ++j) {
            cum += sc[cand[j]];
            if (cum > u * total) {
                pick = cand[j];
                break;
            }
        }
    }
    return pick;
}

int pfo_aco_select(const double sc[8], const uint8_t open[8], uint64_t seed, uint32_t step, uint64_t agent) {
    if (open[0]) return 0;
    return pfo_aco_select_u(sc, open, pfo_uniform(seed, step, PFO_ACO_SELECT, agent, 0));
}

/* ----------------------------------------------------------------- config */

/* src/config.cpp:101-124 (numeric rules only). */
int pfo_validate(const pfo_config* c) {
    if (c->width < 16 || c->width % 16 != 0) return 2;
    if (c->height < 16 || c->height % 16 != 0) return 2;
    if (c->agents_per_side < 0) return 2;
    if (!(c->d0 > 1.0)) return 2;
    if (!(c->sel_sigma >= 0.0)) return 2;
    if (!(c->alpha >= 0.0)) return 2;
    if (!(c->beta >= 0.0)) return 2;
    if (!(c->rho > 0.0 && c->rho <= 1.0)) return 2;
    if (!(c->tau0 > 0.0)) return 2;
    if (!(c->q > 0.0)) return 2;
    const int64_t cells = (int64_t)c->width * c->height;
    if (2 * (int64_t)c->agents_per_side > cells) return 2;
    const int band = pfo_band_height(c->agents_per_side, c->width);
    if (2 * band > c->height) return 2;
    return 0;
}

/* ------------------------------------------------------------ environment */

/* Keyed Fisher-Yates over the band's cell list (src/state.cpp:17-50). */
static int place_side(pfo_state* s, int group, int row_begin, int row_end, int n, uint32_t first_id,
                      uint64_t seed) {
    const size_t m = (size_t)(row_end - row_begin) * (size_t)s->width;
    if (m == 0) return 0;
    size_t* cells = (size_t*)malloc(m * sizeof(size_t));
    if (!cells) return 5;
    size_t t = 0;
    for (int r = row_begin; r < row_end; ++r)
        for (int c = 0; c < s->width; ++c) cells[t++] = (size_t)r * s->width + c;
    for (size_t i = 0; i + 1 < m; ++i) {
        const double u = pfo_uniform(seed, 0, PFO_PLACEMENT, (uint64_t)group, (uint32_t)i);
        size_t off = (size_t)(u * (double)(m - i));
        if (off > m - i - 1) off = m - i - 1;
        const size_t j = i + off;
        const size_t tmp = cells[i];
        cells[i] = cells[j];
        cells[j] = tmp;
    }
    for (int k = 0; k < n; ++k) {
        const size_t cell = cells[k];
        const uint32_t id = first_id + (uint32_t)k;
        const int r = (int)(cell / (size_t)s->width), c = (int)(cell % (size_t)s->width);
        s->occ[cell] = (uint8_t)group;
        s->index[cell] = id;
        pfo_agent* a = &s->agents[id - 1];
        memset(a, 0, sizeof *a);
        a->index = id;
        a->group = (uint8_t)group;
        a->row = a->future_row = r;
        a->col = a->future_col = c;
        a->tour_length = 0.0;
        a->crossed = 0;
    }
    free(cells);
    return 0;
}

/* src/state.cpp:54-75 */
int pfo_new_environment(const pfo_config* cfg, uint64_t seed, pfo_state* s) {
    const int w = cfg->width, h = cfg->height, n = cfg->agents_per_side;
    const int band = pfo_band_height(n, w);
    if (2 * (int64_t)n > (int64_t)w * h || 2 * band > h) return 2;
    const size_t cells = (size_t)w * h;
    s->width = w;
    s->height = h;
    s->model = cfg->model;
    s->n_agents = 2u * (uint32_t)n;
    s->step = 0;
    memset(s->occ, 0, cells);
    memset(s->index, 0, cells * 4);
    memset(s->agents, 0, (size_t)s->n_agents * sizeof(pfo_agent));
    if (cfg->model == PFO_ACO) {
        for (size_t i = 0; i < cells; ++i) s->tau_top[i] = cfg->tau0;
        for (size_t i = 0; i < cells; ++i) s->tau_bot[i] = cfg->tau0;
    }
    int rc = place_side(s, PFO_TOP, 0, band, n, 1, seed);
    if (rc) return rc;
    return place_side(s, PFO_BOTTOM, h - band, h, n, (uint32_t)n + 1, seed);
}

/* --------------------------------------------------------------- the step */

typedef struct engine_consts {
    double dtab[8], eta[8];
    double factor; /* 1 - rho, host-side as src/engine.cpp:126 */
    double diag;   /* kDiagonalStep = sqrt(2), src/aco.cpp:11 */
    int band;
} engine_consts;

static int make_consts(const pfo_config* cfg, engine_consts* k) {
    if (pfo_distance_table(cfg->d0, k->dtab)) return 2;
    for (int i = 0; i < 8; ++i) k->eta[i] = pow(1.0 / k->dtab[i], cfg->beta); /* src/aco.cpp:20-27 */
    k->factor = 1.0 - cfg->rho;
    k->diag = sqrt(2.0);
    k->band = pfo_band_height(cfg->agents_per_side, cfg->width);
    return 0;
}

/* Generic view of a row window so the full-grid step and the cell-resident
 * window step share one implementation. Row indices are global; local buffer
 * row = global row - row0. */
typedef struct view {
    int W, H, row0, nrows;
    uint8_t* occ;
    uint32_t* index;
    double* tau_top;
    double* tau_bot;
} view;

static int v_in_bounds(const view* v, int r, int c) {
    return r >= 0 && r < v->H && c >= 0 && c < v->W && r >= v->row0 && r < v->row0 + v->nrows;
}
static size_t v_at(const view* v, int r, int c) { return (size_t)(r - v->row0) * v->W + c; }

/* neighborhood() (src/grid.cpp:29-40): out-of-bounds slots are walls. */
static void neighborhood(const view* v, const pfo_agent* a, int nr[8], int nc[8], uint8_t open[8]) {
    const int sign = (a->group == PFO_BOTTOM) ? -1 : 1;
    for (int i = 0; i < 8; ++i) {
        nr[i] = a->row + sign * kGoal[i][0];
        nc[i] = a->col + sign * kGoal[i][1];
        open[i] = (uint8_t)(v_in_bounds(v, nr[i], nc[i]) && v->occ[v_at(v, nr[i], nc[i])] == PFO_EMPTY);
    }
}

/* score_phase + intention_phase for one agent (src/engine.cpp:64-90). */
static void intend(const view* v, const pfo_config* cfg, const engine_consts* k, uint64_t seed, uint32_t step,
                   pfo_agent* a) {
    int nr[8], nc[8];
    uint8_t open[8];
    double sc[8];
    neighborhood(v, a, nr, nc, open);
    int pick;
    if (cfg->model == PFO_LEM) {
        pfo_lem_scores(open, k->dtab, sc);
        pick = pfo_lem_select(sc, open, seed, step, a->index, cfg->sel_mu, cfg->sel_sigma);
    } else {
        double tau[8];
        const double* field = (a->group == PFO_TOP) ? v->tau_top : v->tau_bot;
        for (int i = 0; i < 8; ++i) tau[i] = open[i] ? field[v_at(v, nr[i], nc[i])] : 0.0;
        pfo_aco_numerators(open, tau, cfg->alpha, k->eta, sc);
        pick = pfo_aco_select(sc, open, seed, step, a->index);
    }
    a->future_row = pick >= 0 ? nr[pick] : a->row;
    a->future_col = pick >= 0 ? nc[pick] : a->col;
}

/* crossed() (src/metrics.cpp:13-16) */
static int crossed_at(int group, int row, int H, int band) {
    return group == PFO_TOP ? row >= H - band : row <= band - 1;
}

/* movement_phase (src/engine.cpp:92-181) restricted to destination rows
 * [lo, hi) (global); writes are applied only inside [wlo, whi). For the
 * full-grid step both ranges are [0, H). agent_of maps an id to its record. */
typedef struct agent_table {
    pfo_agent* rec;      /* indexable by slot */
    uint32_t* slot_of;   /* id -> slot+1, or NULL for direct agents[id-1] */
} agent_table;

static pfo_agent* agent_by_id(const agent_table* t, uint32_t id) {
    if (!t->slot_of) return &t->rec[id - 1];
    const uint32_t s = t->slot_of[id];
    return s ? &t->rec[s - 1] : NULL;
}

static void movement(const view* v, const pfo_config* cfg, const engine_consts* k, uint64_t seed,
                     uint32_t step, agent_table* at, int lo, int hi, int wlo, int whi, uint32_t* winners,
                     double* tour_cells, uint32_t* cell_words, pfo_report* rep) {
    const int W = v->W;
    /* gather (src/engine.cpp:101-122): winners indexed by local cell */
    for (int r = lo; r < hi; ++r) {
        for (int c = 0; c < W; ++c) {
            const size_t li = v_at(v, r, c);
            winners[li] = 0;
            if (v->occ[li] != PFO_EMPTY) continue;
            uint32_t cont[8];
            int kc = 0;
            for (int j = 0; j < 8; ++j) {
                const int rr = r + kCellNb[j][0], cc = c + kCellNb[j][1];
                if (!v_in_bounds(v, rr, cc)) continue;
                const uint32_t id = v->index[v_at(v, rr, cc)];
                if (id == 0) continue;
                const pfo_agent* a = agent_by_id(at, id);
                if (a && a->future_row == r && a->future_col == c) cont[kc++] = id;
            }
            if (kc == 0) continue;
            const uint64_t gidx = (uint64_t)r * (uint64_t)W + (uint64_t)c;
            const double u = pfo_uniform(seed, step, PFO_RESOLVE, gidx, 0);
            int j = (int)(u * kc);
            if (j > kc - 1) j = kc - 1;
            winners[li] = cont[j];
        }
    }
    /* evaporate (src/engine.cpp:124-131, src/aco.cpp:95-105) */
    if (cfg->model == PFO_ACO) {
        for (int r = wlo; r < whi; ++r)
            for (int c = 0; c < W; ++c) {
                const size_t li = v_at(v, r, c);
                v->tau_top[li] *= k->factor;
                v->tau_bot[li] *= k->factor;
            }
    }
    /* commit (src/engine.cpp:137-175) */
    uint32_t moved = 0, ntop = 0, nbot = 0;
    for (int r = lo; r < hi; ++r) {
        for (int c = 0; c < W; ++c) {
            const size_t li = v_at(v, r, c);
            const uint32_t id = winners[li];
            if (id == 0) continue;
            pfo_agent* a = agent_by_id(at, id);
            const int dr = r - a->row, dc = c - a->col;
            const int dst_in = r >= wlo && r < whi;
            const int src_in = a->row >= wlo && a->row < whi;
            const size_t si = v_at(v, a->row, a->col);
            double tour_src = tour_cells ? tour_cells[si] : a->tour_length;
            if (src_in) {
                v->occ[si] = PFO_EMPTY;
                v->index[si] = 0;
                if (cell_words) cell_words[si] = 0;
            }
            if (!dst_in) continue; /* the owner of the destination commits it */
            v->occ[li] = a->group;
            v->index[li] = id;
            a->row = r;
            a->col = c;
            ++moved;
            if (cfg->model == PFO_ACO) {
                a->tour_length = tour_src + ((dr != 0 && dc != 0) ? k->diag : 1.0);
                double* field = (a->group == PFO_TOP) ? v->tau_top : v->tau_bot;
                field[li] += cfg->q / a->tour_length; /* deposit, src/aco.cpp:119-123 */
                if (tour_cells) tour_cells[li] = a->tour_length;
            }
            if (!a->crossed && crossed_at(a->group, r, v->H, k->band)) {
                a->crossed = 1;
                if (a->group == PFO_TOP) ++ntop;
                else ++nbot;
            }
            if (cell_words)
                cell_words[li] = id | ((uint32_t)a->crossed << 29) | ((uint32_t)a->group << 30);
        }
    }
    rep->step = step;
    rep->moved = moved;
    rep->newly_crossed_top = ntop;
    rep->newly_crossed_bottom = nbot;
}

/* StepEngine::step (src/engine.cpp:53-62) */
int pfo_step(pfo_state* s, const pfo_config* cfg, uint64_t seed, pfo_report* out) {
    engine_consts k;
    if (make_consts(cfg, &k)) return 2;
    view v = {s->width, s->height, 0, s->height, s->occ, s->index, s->tau_top, s->tau_bot};
    for (uint32_t i = 0; i < s->n_agents; ++i) intend(&v, cfg, &k, seed, s->step, &s->agents[i]);
    uint32_t* winners = (uint32_t*)malloc((size_t)s->width * s->height * 4);
    if (!winners) return 5;
    agent_table at = {s->agents, NULL};
    pfo_report rep;
    movement(&v, cfg, &k, seed, s->step, &at, 0, s->height, 0, s->height, winners, NULL, NULL, &rep);
    free(winners);
    /* reset_phase (src/engine.cpp:183-193) */
    for (uint32_t i = 0; i < s->n_agents; ++i) {
        s->agents[i].future_row = s->agents[i].row;
        s->agents[i].future_col = s->agents[i].col;
    }
    ++s->step;
    if (out) *out = rep;
    return 0;
}

int pfo_run(pfo_state* s, const pfo_config* cfg, uint64_t seed, uint32_t n, pfo_report* out) {
    for (uint32_t i = 0; i < n; ++i) {
        const int rc = pfo_step(s, cfg, seed, out ? &out[i] : NULL);
        if (rc) return rc;
    }
    return 0;
}

/* Cell-resident window step: rebuild agent records from the cell words of the
 * local buffer, run one reference step over it, and write back only rows
 * [lo, hi). */
int pfo_step_cells(const pfo_config* cfg, uint64_t seed, uint32_t step, int32_t row0, int32_t nrows,
                   uint32_t* cell, double* tour, double* tau_top, double* tau_bot, int32_t lo, int32_t hi,
                   pfo_report* out) {
    engine_consts k;
    if (make_consts(cfg, &k)) return 2;
    const int W = cfg->width;
    const size_t n = (size_t)nrows * W;
    uint8_t* occ = (uint8_t*)calloc(n, 1);
    uint32_t* index = (uint32_t*)calloc(n, 4);
    uint32_t* winners = (uint32_t*)calloc(n, 4);
    const uint32_t max_id = 2u * (uint32_t)cfg->agents_per_side;
    uint32_t* slot_of = (uint32_t*)calloc((size_t)max_id + 1, 4);
    pfo_agent* rec = (pfo_agent*)calloc(n ? n : 1, sizeof(pfo_agent));
    if (!occ || !index || !winners || !slot_of || !rec) return 5;
    uint32_t na = 0;
    for (int lr = 0; lr < nrows; ++lr) {
        const int g = row0 + lr;
        for (int c = 0; c < W; ++c) {
            const size_t li = (size_t)lr * W + c;
            const uint32_t w = cell[li];
            if (g < 0 || g >= cfg->height || w == 0) continue;
            const uint32_t id = w & 0x1FFFFFFFu;
            pfo_agent* a = &rec[na];
            a->index = id;
            a->group = (uint8_t)(w >> 30);
            a->row = a->future_row = g;
            a->col = a->future_col = c;
            a->crossed = (uint8_t)((w >> 29) & 1u);
            a->tour_length = tour ? tour[li] : 0.0;
            occ[li] = a->group;
            index[li] = id;
            slot_of[id] = ++na;
        }
    }
    view v = {W, cfg->height, row0, nrows, occ, index, tau_top, tau_bot};
    /* Intentions for every agent present; those far from [lo, hi) are unused. */
    for (uint32_t i = 0; i < na; ++i) intend(&v, cfg, &k, seed, step, &rec[i]);
    agent_table at = {rec, slot_of};
    pfo_report rep;
    int glo = row0 + lo - 1, ghi = row0 + hi + 1; /* gather destinations one row beyond */
    if (glo < row0) glo = row0;
    if (ghi > row0 + nrows) ghi = row0 + nrows;
    /* movement writes cell words only inside the window */
    movement(&v, cfg, &k, seed, step, &at, glo, ghi, row0 + lo, row0 + hi, winners, tour, cell, &rep);
    free(occ);
    free(index);
    free(winners);
    free(slot_of);
    free(rec);
    if (out) *out = rep;
    return 0;
}

/* ----------------------------------------------------------------- hashes */

uint64_t pfo_fnv1a(const void* data, uint64_t n, uint64_t h) {
    const uint8_t* p = (const uint8_t*)data;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

#define FNV_OFFSET 0xcbf29ce484222325ull

uint64_t pfo_hash_index(const pfo_state* s) {
    return pfo_fnv1a(s->index, (uint64_t)s->width * s->height * 4, FNV_OFFSET);
}
uint64_t pfo_hash_occ(const pfo_state* s) {
    return pfo_fnv1a(s->occ, (uint64_t)s->width * s->height, FNV_OFFSET);
}
uint64_t pfo_hash_agents(const pfo_state* s) {
    uint64_t h = FNV_OFFSET;
    for (uint32_t i = 0; i < s->n_agents; ++i) {
        const pfo_agent* a = &s->agents[i];
        h = pfo_fnv1a(&a->row, 4, h);
        h = pfo_fnv1a(&a->col, 4, h);
        h = pfo_fnv1a(&a->tour_length, 8, h);
        h = pfo_fnv1a(&a->crossed, 1, h);
    }
    return h;
}
uint64_t pfo_hash_pher(const pfo_state* s) {
    const uint64_t n = (uint64_t)s->width * s->height * 8;
    return pfo_fnv1a(s->tau_bot, n, pfo_fnv1a(s->tau_top, n, FNV_OFFSET));
}
uint64_t pfo_hash_series(const pfo_report* r, uint32_t n) {
    return pfo_fnv1a(r, (uint64_t)n * sizeof(pfo_report), FNV_OFFSET);
}
