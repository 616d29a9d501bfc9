/*
 * fleetplace_b200.h — C ABI of the B200-native fleet-placement hot path.
 *
 * This is the drop-in boundary for the reference's solver path
 *   build_distance_table  -> rank_bases -> tabu_search / local_search
 * (reference `fleetplace`, /root/reference/proj/include/fleetplace/*.hpp).
 * Every entry point is `extern "C"`, takes plain pointers and sizes, and
 * never exposes CUDA or torch types. A C++ adapter or the
 * Python mirror (paper_2001_05291_b200/fleetplace.py) converts the
 * reference's id-keyed `Assignment` maps to the index arrays used here.
 *
 * Conventions
 *  - Entities are addressed by INDEX in instance (load) order, as the
 *    reference's SearchState does (proj/src/search_state.hpp:20-31). Ids are
 *    carried only where the reference's semantics depend on them (tie breaks
 *    by base id, vehicle-id ordering of the initial pool, the shared
 *    {MoveKind, id} tabu key space).
 *  - The distance table is missions x bases, fp64, column-major: entry
 *    (m, b) at b * n_missions + m, exactly Eigen's default layout used by
 *    DistanceTable::cost (proj/include/fleetplace/model.hpp:63-66).
 *  - Every call is synchronous at return. A context is not thread-safe; use
 *    one per host thread (the reference's entry points are reentrant because
 *    they keep no globals, proj/src/search.cpp:401-434).
 *  - Errors: functions return an fp_status; fp_last_error() returns the
 *    message of the most recent failure on the calling thread. Status codes
 *    map 1:1 onto the exception types the reference throws
 *    (proj/include/fleetplace/errors.hpp:8-62, std::invalid_argument,
 *    std::logic_error).
 */
#ifndef FLEETPLACE_B200_H_
#define FLEETPLACE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP_ABI_VERSION 4

typedef enum fp_status {
  FP_OK = 0,
  FP_ERR_INVALID_ARGUMENT = 1,   /* std::invalid_argument                 */
  FP_ERR_VALIDATION = 2,         /* fleetplace::ValidationError           */
  FP_ERR_INFEASIBLE = 3,         /* fleetplace::InfeasibleError           */
  FP_ERR_NO_COMPATIBLE = 4,      /* fleetplace::NoCompatibleVehicleError  */
  FP_ERR_POOL_TOO_SMALL = 5,     /* fleetplace::PoolTooSmallError         */
  FP_ERR_LOGIC = 6,              /* std::logic_error (delta drift)        */
  FP_ERR_ERROR = 7,              /* fleetplace::Error (generic)           */
  FP_ERR_CUDA = 8,               /* CUDA runtime failure / no device      */
  FP_ERR_OUT_OF_MEMORY = 9
} fp_status;

/* BaseKind / VehicleKind / PoolEntryKind / SearchMode / MoveKind, with the
 * reference's enumerator order (model.hpp:12-13, search.hpp:14-32). */
enum { FP_AERODROME = 0, FP_HELIPAD = 1 };
enum { FP_ROTARY = 0, FP_FIXED = 1 };
enum { FP_POOL_EMPTY_BASE = 0, FP_POOL_IDLE_VEHICLE = 1 };
enum { FP_MODE_LOCAL = 0, FP_MODE_TABU = 1 };
enum { FP_MOVE_TAKEOVER = 0, FP_MOVE_RELOCATE = 1, FP_MOVE_REASSIGN = 2 };

/* Instance in structure-of-arrays form (proj/include/fleetplace/model.hpp:15-54).
 * All arrays are host memory owned by the caller. */
typedef struct fp_instance {
  int32_t n_bases;
  const int32_t* base_id;
  const uint8_t* base_kind;      /* FP_AERODROME | FP_HELIPAD */
  const double* base_lat;
  const double* base_lon;
  int32_t n_vehicles;
  const int32_t* vehicle_id;
  const uint8_t* vehicle_kind;   /* FP_ROTARY | FP_FIXED */
  int32_t n_missions;
  const int32_t* mission_id;
  const double* pickup_lat;
  const double* pickup_lon;
  const double* delivery_lat;
  const double* delivery_lon;
  const uint8_t* rotary_only;    /* 0 | 1 */
} fp_instance;

/* SearchConfig (proj/include/fleetplace/search.hpp:16-26). */
typedef struct fp_search_config {
  uint64_t seed;
  int32_t mode;                  /* FP_MODE_LOCAL | FP_MODE_TABU */
  int32_t tabu_tenure;           /* 0 = auto (2 x missions), < 0 rejected */
  int32_t max_passes;            /* < 0 = no cap (std::nullopt) */
  int32_t debug_check_deltas;    /* non-zero: verify the total after every move */
} fp_search_config;

/* SearchStats (proj/include/fleetplace/search.hpp:68-76). */
typedef struct fp_search_stats {
  uint64_t passes;
  uint64_t evaluations;
  uint64_t applied_moves;
  uint64_t committed_moves;
  uint64_t tabu_skips_outer;
  uint64_t tabu_skips_inner;
  double final_objective_km;
} fp_search_stats;

/* Search start: an Assignment plus the UnusedPool, in index form.
 * vehicle_base[v]   = base index of vehicle v, or -1 if unplaced
 * mission_vehicle[m]= serving vehicle index of mission m, or -1 if unserved
 * pool_kind/pool_index: the UnusedPool entries in order (search.hpp:34-49);
 *   pool_index holds a base index (EMPTY_BASE) or a vehicle index
 *   (IDLE_VEHICLE); -1 stands for an id the instance does not know. */
typedef struct fp_search_start {
  const int32_t* vehicle_base;
  const int32_t* mission_vehicle;
  int32_t pool_size;
  const int32_t* pool_kind;
  const int32_t* pool_index;
} fp_search_start;

/* Search result: the final Assignment in index form plus SearchStats. */
typedef struct fp_search_result {
  int32_t* vehicle_base;         /* [n_vehicles] */
  int32_t* mission_vehicle;      /* [n_missions] */
  fp_search_stats stats;
  double device_ms;              /* CUDA-event time of the device search */
  uint64_t kernel_launches;      /* kernels this call launched */
  uint64_t exact_fallbacks;      /* accept decisions settled by exact chains */
  uint64_t phase_cycles[16];     /* SM cycles per automaton phase (scenario 0):
                                    row runs, row context, scan steps, event
                                    pairs, exact fallbacks, table-row rebuilds,
                                    relocation bit updates, substitution bit
                                    updates, relocation apply, exact totals,
                                    table patches, per-pass setup, exact
                                    relocation deltas, exact candidate totals,
                                    helper waits, (reserved); all zero unless
                                    the library is built with -DFP_PHASE_CLOCKS
                                    (a profiling build: the clocks cost ~5%) */
  double init_ms;                /* search start: costs, exact total, relocation
                                    table sweep (CUDA events) */
  double sweep_ms;               /* per-pass bitset sweeps (grid-wide mode) */
  uint64_t event_counts[5];      /* scenario 0: scanned rows, scan steps, row
                                    contexts, table-row rebuilds, rows settled
                                    by the O(1) eventless test */
  double init_part_ms[4];        /* init_ms split: row-major table copy, costs +
                                    exact total, improvement rows, relocation
                                    table rows (CUDA events) */
  double pass_ms;                /* pass-kernel launches (CUDA events, summed) */
  uint64_t pass_launches;        /* pass-kernel launches of this call */
} fp_search_result;

/* RankedStart (proj/include/fleetplace/rank.hpp:10-14) in index form. */
typedef struct fp_ranked_start {
  double* base_totals;           /* [n_bases]  fixed-order column sums */
  int32_t* vehicle_base;         /* [n_vehicles] base index */
  int32_t* mission_vehicle;      /* [n_missions] vehicle index */
  int32_t* unused_bases;         /* [n_bases]  base indices, ranking order */
  int32_t n_unused;              /* out */
} fp_ranked_start;

typedef struct fp_ctx fp_ctx;

/* ---- library / context ------------------------------------------------- */
int32_t fp_abi_version(void);
const char* fp_last_error(void);
/* Opens `device` (CUDA ordinal) and creates a stream + device workspace. */
fp_status fp_ctx_create(int32_t device, fp_ctx** out);
void fp_ctx_destroy(fp_ctx* ctx);
/* Kernel launches issued by this context since creation (evidence counter). */
uint64_t fp_ctx_kernel_launches(const fp_ctx* ctx);
/* CUDA-event time of the main kernel of the last fp_build_distance_table /
 * fp_column_totals / fp_rank_bases call on this context (ms). */
double fp_ctx_last_kernel_ms(const fp_ctx* ctx);
/* CUDA-event time of the last row-major copy of the resident table (made on
 * the context's second stream after fp_build_distance_table /
 * fp_table_upload; waits for it), or 0 if none was made. */
double fp_ctx_last_copy_ms(fp_ctx* ctx);
/* (new; no reference counterpart) enabled != 0 (the default): every
 * fp_build_distance_table / fp_table_upload starts the row-major copy of the
 * table on the context's second stream, ready for the next fp_search.
 * 0: no eager copy -- a table that is only ranked (a mission shard whose
 * search runs elsewhere) skips it; a later fp_search on the context makes
 * the copy itself, in-stream. Results never depend on it. */
fp_status fp_ctx_set_row_copy(fp_ctx* ctx, int32_t enabled);

/* The search's permutation stream (perm_a, perm_b of every pass: std::
 * mt19937_64(seed), Fisher-Yates with uniform_below; proj/src/search.cpp:
 * 401-413) drawn on the device: 2*passes permutations of n into out
 * [2*passes*n]. Used by searches whose passes run in one launch; exposed for
 * tests. n >= 2. */
fp_status fp_permutations(fp_ctx* ctx, uint64_t seed, int32_t n, int32_t passes, int32_t* out);

/* ---- instance validation / generation (host) -------------------------- */
/* validate_instance (proj/src/model.cpp:46-74). */
fp_status fp_validate_instance(const fp_instance* inst);

/* synthesize_pool + generate_instance (proj/src/data.cpp:110-180) with the
 * default PoolShape; `bbox` = {lat_min, lat_max, lon_min, lon_max} or NULL
 * for BoundingBox{}. Output arrays are caller-allocated with sizes
 * n_bases = aerodromes + helipads, n_vehicles = rotary + fixed,
 * n_missions = missions. Deterministic per seed (same libm => same bits). */
fp_status fp_generate_instance(uint64_t pool_seed, const double* bbox,
                               int32_t aerodromes, int32_t helipads,
                               int32_t health_sites, int32_t missions,
                               double rotary_only_fraction, uint64_t seed,
                               int32_t rotary, int32_t fixed_wing,
                               int32_t* base_id, uint8_t* base_kind,
                               double* base_lat, double* base_lon,
                               int32_t* vehicle_id, uint8_t* vehicle_kind,
                               int32_t* mission_id, double* pickup_lat,
                               double* pickup_lon, double* delivery_lat,
                               double* delivery_lon, uint8_t* rotary_only);

/* ---- kernel (1): distance table ---------------------------------------- */
/* build_distance_table (proj/src/model.cpp:76-90): builds the missions x
 * bases table on the device; it stays resident in `ctx` for the calls
 * below. `out_cost` (host, n_missions*n_bases) may be NULL. */
fp_status fp_build_distance_table(fp_ctx* ctx, const fp_instance* inst,
                                  double radius_km, double* out_cost);
/* Makes a caller-supplied table (e.g. the reference's) resident instead.
 * Any matrix is accepted (column totals are exact for every entry value,
 * like the reference's loop); fp_search additionally requires every entry to
 * be finite and >= 0, as distances are, and returns FP_ERR_INVALID_ARGUMENT
 * otherwise (one device pass checks the upload). */
fp_status fp_table_upload(fp_ctx* ctx, int32_t n_missions, int32_t n_bases,
                          const double* cost_colmajor);
fp_status fp_table_download(fp_ctx* ctx, double* out_cost);

/* haversine_km / mission_cost_km (proj/include/fleetplace/geo.hpp:22-30) on
 * n point pairs with kernel (1)'s arithmetic: out[k] = hav(a_k, b_k) +
 * (c_lat ? hav(a_k, c_k) : 0). Host arrays; c_lat/c_lon may be NULL. */
fp_status fp_haversine_batch(fp_ctx* ctx, int32_t n, const double* a_lat,
                             const double* a_lon, const double* b_lat,
                             const double* b_lon, const double* c_lat,
                             const double* c_lon, double radius_km, double* out);

/* ---- kernel (2): ranking ------------------------------------------------ */
/* column_totals (proj/src/rank.cpp:10-23): out[b] = sum_m cost(m, b) in row
 * order, bit-identical to the sequential reference. */
fp_status fp_column_totals(fp_ctx* ctx, double* out_totals);
/* rank_bases (proj/src/rank.cpp:25-124) on the resident table. */
fp_status fp_rank_bases(fp_ctx* ctx, const fp_instance* inst,
                        fp_ranked_start* out);

/* ---- missions sharded across GPUs ---------------------- */
/* A mission shard's context holds the table of a contiguous mission range
 * (fp_build_distance_table / fp_table_upload on an instance carrying all
 * bases and vehicles and that range's missions).
 *
 * column_totals (proj/src/rank.cpp:10-23) continued across shards: for the
 * columns [b0, b0 + nb), out[k] = the fixed-order fp64 chain over this
 * shard's rows starting at carry[k] (NULL: 0.0). Feeding shard g's `out` as
 * shard g+1's `carry` gives, on the last shard, the reference's totals bit
 * for bit (the sum is never reassociated; rank.hpp:16-18's bit-identity
 * contract). device_ptrs = 1: carry/out are device pointers on ctx's device
 * (e.g. NCCL buffers), 0: host pointers. Synchronous at return. */
fp_status fp_column_totals_chain(fp_ctx* ctx, int32_t b0, int32_t nb,
                                 const double* carry, double* out,
                                 int32_t device_ptrs);
/* rank_bases steps (2)-(6) (proj/src/rank.cpp:35-121) from given totals of
 * all bases (host, n_bases): rank order, helipad cap, placement, and the
 * per-mission argmin for the resident table's missions (those of `inst`,
 * e.g. one shard). out->base_totals receives a copy of totals. */
fp_status fp_rank_from_totals(fp_ctx* ctx, const fp_instance* inst,
                              const double* totals, fp_ranked_start* out);

/* ---- kernels (3)+(4): search ------------------------------------------- */
/* initial_pool (proj/src/search.cpp:364-377): unused bases in the given
 * order, then placed vehicles serving no mission, in vehicle-id order.
 * out_kind/out_index need room for n_unused + n_vehicles entries. */
fp_status fp_initial_pool(const fp_instance* inst, const int32_t* vehicle_base,
                          const int32_t* mission_vehicle,
                          const int32_t* unused_bases, int32_t n_unused,
                          int32_t* out_kind, int32_t* out_index,
                          int32_t* out_size);

/* tabu_search / local_search (proj/src/search.cpp:438-460) on the resident
 * table: same Assignment and same SearchStats as the reference. */
fp_status fp_search(fp_ctx* ctx, const fp_instance* inst,
                    const fp_search_config* cfg, const fp_search_start* start,
                    fp_search_result* out);

/* Scenario batch: `n` independent searches of one mission count (tables
 * uploaded or built per scenario into the batch arena), run concurrently,
 * one thread block per scenario, each with its OWN SearchConfig cfgs[s]
 * (seed, mode, tenure, max_passes, debug): e.g. run_experiment's attempts,
 * attempt t searching the same instance with seed + t
 * (proj/src/bench.cpp:125-128), or independent scenarios. Scenario s's
 * result equals fp_search's on its own. Scenarios with equal seeds share one
 * permutation stream (it depends on the seed and n_missions only).
 * tables[s] (or tables itself) may be NULL: scenario s's table is then built
 * on the device by kernel (1) with radius_km (all such tables in one
 * launch); the context's resident table is never touched. (new; the
 * reference runs attempts one after another) */
fp_status fp_search_batch_configs(fp_ctx* ctx, int32_t n, const fp_instance* insts,
                                  const double* const* tables, double radius_km,
                                  const fp_search_config* cfgs,
                                  const fp_search_start* starts,
                                  fp_search_result* outs);
/* The same with one config for every scenario and radius 6371.0088. */
fp_status fp_search_batch(fp_ctx* ctx, int32_t n, const fp_instance* insts,
                          const double* const* tables,
                          const fp_search_config* cfg,
                          const fp_search_start* starts,
                          fp_search_result* outs);

/* (new; SURVEY.md §8(d)'s roofline kernel, exposed for mission-sharded use,
 * §8(e)) The neighbourhood sweep of a search start on the resident table:
 * every relocation's quick delta to every base and every reassignment /
 * takeover's improvement test, as the search computes them before its first
 * pass. With a mission shard (the instance and start of one mission range,
 * all bases and vehicles) it is the shard's PARTIAL sweep: the relocation
 * sums of all shards add up (sharded.neighbourhood_sweep_sharded combines
 * them with one NCCL all-reduce, widening the error bound by the additions),
 * the improvement rows and mission costs concatenate. */
typedef struct fp_sweep_result {
  double* reloc_sum;        /* [n_vehicles * n_bases] entry (t, v) at v*n_bases + t:
                               any-order sum over v's missions m of
                               cost(m, t) - mc[m] (eval_relocate's quick delta,
                               proj/src/search.cpp:121-127, as a real sum) */
  double* reloc_err;        /* [..] |reloc_sum - exact real sum| <= reloc_err */
  double* reloc_abs;        /* [..] >= sum |cost(m, t) - mc[m]| */
  uint32_t* improve_rows;   /* [n_missions * ceil(n_vehicles / 32)]: bit g of row m
                               = moving m to vehicle g lowers its cost
                               (eval_reassign / eval_takeover, search.cpp:82-148) */
  double* mission_cost;     /* [n_missions] mc[m] = cost(m, base of m's vehicle) */
  int32_t device_ptrs;      /* 1: the outputs are device pointers on ctx's device */
  double sweep_ms;          /* CUDA events: improvement rows + relocation sums */
  double total_ms;          /* ... plus mission costs and the exact start total */
} fp_sweep_result;
fp_status fp_neighbourhood_sweep(fp_ctx* ctx, const fp_instance* inst,
                                 const fp_search_start* start, fp_sweep_result* out);

/* enumerate_moves (proj/src/search.cpp:379-397): the up-to-three proposals
 * reachable from (i, j) with their exact fixed-order deltas. Outputs kind
 * and delta arrays with room for 3 entries. */
fp_status fp_enumerate_moves(fp_ctx* ctx, const fp_instance* inst,
                             const fp_search_start* state, int32_t i,
                             int32_t j_mission_index, int32_t* out_kind,
                             double* out_delta, int32_t* out_count);

/* objective_km's fixed mission-order sum (proj/src/model.cpp:176-192) of
 * cost(m, vehicle_base[mission_vehicle[m]]) on the resident table.
 * Full feasibility (check_feasible) is the caller's; here every
 * mission_vehicle[m] must be in [0, n_vehicles) and every referenced
 * vehicle_base in [0, n_bases), else FP_ERR_INFEASIBLE. */
fp_status fp_objective_km(fp_ctx* ctx, int32_t n_vehicles, const int32_t* vehicle_base,
                          const int32_t* mission_vehicle, double* out_km);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* FLEETPLACE_B200_H_ */
