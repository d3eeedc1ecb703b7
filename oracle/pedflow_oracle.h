/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference hot path (the per-time-step grid update
 * of /root/reference/proj, "pedflow"). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load liboracle.so, and only as the checker.
 *
 * Parity pinned by: the Random123 Philox4x32-10 known-answer vectors, the SPEC
 * per-operation examples, the
 * FNV-1a anchors of SURVEY.md §8(c) (tests/golden/anchors.json), and
 * differential runs against oracle/_ref (the reference compiled from its own
 * sources) — see tests/test_oracle.py.
 */
#ifndef PEDFLOW_ORACLE_H
#define PEDFLOW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PFO_EMPTY = 0, PFO_TOP = 1, PFO_BOTTOM = 2 };
enum { PFO_LEM = 0, PFO_ACO = 1 };
enum { PFO_PLACEMENT = 0, PFO_LEM_SELECT = 1, PFO_ACO_SELECT = 2, PFO_RESOLVE = 3, PFO_TIE_BREAK = 4 };

/* Numeric part of ScenarioConfig (inc/config.hpp:20-58). */
typedef struct pfo_config {
    int32_t width, height, agents_per_side, model;
    uint64_t seed;
    double d0, sel_mu, sel_sigma, alpha, beta, rho, tau0, q;
} pfo_config;

/* Byte-identical to AgentRecord (inc/grid.hpp:84-93): 40 bytes. */
typedef struct pfo_agent {
    uint32_t index;
    uint8_t group;
    int32_t row, col, future_row, future_col;
    double tour_length;
    uint8_t crossed;
} pfo_agent;

/* StepReport (inc/engine.hpp:16-21). */
typedef struct pfo_report {
    uint32_t step, moved, newly_crossed_top, newly_crossed_bottom;
} pfo_report;

/* The SimState planes (inc/state.hpp:16-31); caller-owned arrays. */
typedef struct pfo_state {
    int32_t width, height, model;
    uint32_t n_agents;
    uint8_t* occ;      /* H*W */
    uint32_t* index;   /* H*W, 0 = empty */
    pfo_agent* agents; /* n_agents, agents[id-1] */
    double* tau_top;   /* H*W, ACO only (may be NULL for LEM) */
    double* tau_bot;
    uint32_t step;
} pfo_state;

uint32_t pfo_agent_size(void);

/* det-rng (src/rng.cpp) */
uint64_t pfo_random_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter);
double pfo_uniform(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter);
double pfo_inverse_normal_cdf(double p);
/* glibc 2.39's log (x86-64 FMA variant) restated op for op, for positive
 * normal x outside [1 - 2^-4, 1 + 0x1.09p-4] (the AS241 tail domain); the
 * checker of the device's pfdev::glibc_log. NaN outside that domain. */
double pfo_log_restated(double x);
/* 1 where this host's log is the variant the restatement follows. */
int pfo_log_restated_matches_host(uint32_t n, uint64_t seed);
/* pfo_normal over arrays of keys (out[i] for key i). */
void pfo_normal_batch(uint32_t n, const uint64_t* seed, const uint32_t* step, const uint32_t* phase,
                      const uint64_t* entity, const uint32_t* counter, double mu, double sigma, double* out);
double pfo_normal(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter,
                  double mu, double sigma);

/* grid-core / policies (src/grid.cpp, src/lem.cpp, src/aco.cpp, src/metrics.cpp) */
int pfo_distance_table(double d0, double out[8]);
int32_t pfo_band_height(int32_t agents_per_side, int32_t width);
/* open[8]: 1 if the goal-relative slot is open. out[8]: scores. */
void pfo_lem_scores(const uint8_t open[8], const double dtable[8], double out[8]);
void pfo_aco_numerators(const uint8_t open[8], const double tau[8], double alpha, const double eta[8],
                        double out[8]);
/* Returns the chosen goal-relative slot 0..7, or -1 for stay. */
int pfo_lem_select(const double scores[8], const uint8_t open[8], uint64_t seed, uint32_t step,
                   uint64_t agent, double mu_sel, double sigma_sel);
int pfo_lem_select_u(const double scores[8], const uint8_t open[8], double r_unclamped, double tie_u);
int pfo_aco_select(const double scores[8], const uint8_t open[8], uint64_t seed, uint32_t step,
                   uint64_t agent);
int pfo_aco_select_u(const double scores[8], const uint8_t open[8], double u);

/* Validation rules of validate() (src/config.cpp:101-124). 0 ok, 2 config error. */
int pfo_validate(const pfo_config* cfg);

/* new_environment (src/state.cpp:17-75). Arrays must be allocated by the
 * caller: occ/index H*W, agents 2n, tau_* H*W (ACO). */
int pfo_new_environment(const pfo_config* cfg, uint64_t seed, pfo_state* s);

/* StepEngine::step (src/engine.cpp:53-193), sequential. */
int pfo_step(pfo_state* s, const pfo_config* cfg, uint64_t seed, pfo_report* out);
int pfo_run(pfo_state* s, const pfo_config* cfg, uint64_t seed, uint32_t n, pfo_report* out);

/* Cell-resident window step (test adapter for the row-sharded N>1 path).
 * The local buffer holds rows [row0, row0+nrows) of a global H x W grid in the
 * product's packed format: cell word = id | crossed<<29 | group<<30, tour f64
 * per cell (valid where occupied), tau_top/tau_bot per cell. Rows outside
 * [0, H) are walls. One reference step is applied, but only cells in local
 * rows [lo, hi) are written and counted; everything else is left stale for the
 * halo exchange to overwrite. Requires 3 valid rows around [lo, hi). */
int pfo_step_cells(const pfo_config* cfg, uint64_t seed, uint32_t step, int32_t row0, int32_t nrows,
                   uint32_t* cell, double* tour, double* tau_top, double* tau_bot, int32_t lo,
                   int32_t hi, pfo_report* out);

/* FNV-1a 64 anchors, as defined in SURVEY.md §8(c). */
uint64_t pfo_fnv1a(const void* data, uint64_t n, uint64_t h);
uint64_t pfo_hash_index(const pfo_state* s);
uint64_t pfo_hash_occ(const pfo_state* s);
uint64_t pfo_hash_agents(const pfo_state* s);
uint64_t pfo_hash_pher(const pfo_state* s);
uint64_t pfo_hash_series(const pfo_report* r, uint32_t n);

#ifdef __cplusplus
}
#endif
#endif
