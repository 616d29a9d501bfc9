/*
 * oracle/fleetplace_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never
 * the product). A plain-C restatement of the reference's hot path:
 *
 *   haversine_km / mission_cost_km     proj/src/geo.cpp:18-36
 *   build_distance_table               proj/src/model.cpp:76-90
 *   column_totals                      proj/src/rank.cpp:10-23
 *   rank_bases                         proj/src/rank.cpp:25-124
 *   initial_pool                       proj/src/search.cpp:364-377
 *   SearchState::from                  proj/src/search.cpp:14-65
 *   eval_takeover/relocate/reassign    proj/src/search.cpp:82-148
 *   candidate_total                    proj/src/search.cpp:150-167
 *   apply_move                         proj/src/search.cpp:169-220
 *   candidate_tabu_keys/outer/inner    proj/src/search.cpp:226-264
 *   try_move / run_row / run_search    proj/src/search.cpp:277-346, 401-434
 *   TabuList                           proj/include/fleetplace/search.hpp:78-122
 *   mt19937_64 + uniform_below + Fisher-Yates
 *                                      proj/include/fleetplace/rng.hpp:14-42,
 *                                      proj/src/rng.cpp:17-22
 *
 * The tabu list is restated in the expiry-stamp form: a
 * key inserted while `tick` pairs have completed lives while tick < expiry,
 * expiry = tick + tenure; re-insertion overwrites role and expiry. This is
 * equivalent to the reference's per-pair decrement_all map.
 *
 * Parity is PINNED against the compiled reference (oracle/_ref/
 * libfleetplace_ref.so, built from the unmodified sources by oracle/Makefile)
 * in tests/test_oracle.py and by the golden fixtures in tests/golden/.
 * Beyond the reference API it can emit a move log (one record per applied
 * move), which the GPU debug path is compared against to locate the first
 * divergence.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fleetplace_b200.h"

static const double kDegToRad = 3.14159265358979323846 / 180.0;

/* ---------------------------------------------------------------- geo ---- */
double or_haversine_km(double lat_a, double lon_a, double lat_b, double lon_b,
                       double radius_km) {
  const double phi_a = lat_a * kDegToRad;
  const double phi_b = lat_b * kDegToRad;
  const double half_dphi = 0.5 * fabs(lat_b - lat_a) * kDegToRad;
  const double half_dpsi = 0.5 * fabs(lon_b - lon_a) * kDegToRad;
  const double s_lat = sin(half_dphi);
  const double s_lon = sin(half_dpsi);
  const double h = s_lat * s_lat + cos(phi_a) * cos(phi_b) * s_lon * s_lon;
  const double r = sqrt(h);
  return 2.0 * radius_km * asin(r < 1.0 ? r : 1.0);
}

double or_mission_cost_km(double blat, double blon, double plat, double plon,
                          double dlat, double dlon, double radius_km) {
  return or_haversine_km(blat, blon, plat, plon, radius_km) +
         or_haversine_km(blat, blon, dlat, dlon, radius_km);
}

void or_build_table(const fp_instance* in, double radius_km, double* out) {
  const int64_t M = in->n_missions;
  for (int b = 0; b < in->n_bases; ++b)
    for (int64_t m = 0; m < M; ++m)
      out[b * M + m] = or_mission_cost_km(in->base_lat[b], in->base_lon[b],
                                          in->pickup_lat[m], in->pickup_lon[m],
                                          in->delivery_lat[m], in->delivery_lon[m],
                                          radius_km);
}

void or_column_totals(int32_t M, int32_t B, const double* cost, double* out) {
  for (int b = 0; b < B; ++b) {
    double s = 0.0;
    for (int64_t m = 0; m < M; ++m) s += cost[(int64_t)b * M + m];
    out[b] = s;
  }
}

/* ---------------------------------------------------------------- rng ---- */
typedef struct {
  uint64_t mt[312];
  int mti;
} or_mt64;

static void mt_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}

static uint64_t mt_next(or_mt64* g) {
  if (g->mti >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static uint64_t uniform_below(or_mt64* g, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  uint64_t x = mt_next(g);
  while (x < threshold) x = mt_next(g);
  return x % n;
}

static void random_permutation(or_mt64* g, int n, int* out) {
  for (int i = 0; i < n; ++i) out[i] = i;
  for (int64_t i = n; i > 1; --i) {
    const int64_t j = (int64_t)uniform_below(g, (uint64_t)i);
    const int t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

/* Exposed for the RNG parity test: writes `count` raw draws. */
void or_mt19937_64(uint64_t seed, int32_t count, uint64_t* out) {
  or_mt64 g;
  mt_seed(&g, seed);
  for (int i = 0; i < count; ++i) out[i] = mt_next(&g);
}

void or_permutations(uint64_t seed, int32_t n, int32_t passes, int32_t* out) {
  or_mt64 g;
  mt_seed(&g, seed);
  for (int p = 0; p < 2 * passes; ++p) random_permutation(&g, n, out + (int64_t)p * n);
}

/* ---------------------------------------------------------------- rank --- */
static const double* g_tot;
static const int32_t* g_bid;
static int cmp_rank(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  if (g_tot[x] != g_tot[y]) return g_tot[x] < g_tot[y] ? -1 : 1;
  return g_bid[x] < g_bid[y] ? -1 : (g_bid[x] > g_bid[y]);
}
static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return x < y ? -1 : (x > y);
}

/* rank_bases minus validate_instance (the tests validate separately).
 * Returns FP_OK, FP_ERR_VALIDATION or FP_ERR_NO_COMPATIBLE. */
int or_rank_bases(const fp_instance* in, const double* cost, fp_ranked_start* out) {
  const int B = in->n_bases, V = in->n_vehicles;
  const int64_t M = in->n_missions;
  or_column_totals((int32_t)M, B, cost, out->base_totals);
  int* order = (int*)malloc(sizeof(int) * (B + 1));
  for (int b = 0; b < B; ++b) order[b] = b;
  g_tot = out->base_totals;
  g_bid = in->base_id;
  qsort(order, (size_t)B, sizeof(int), cmp_rank);
  int rotary = 0;
  for (int v = 0; v < V; ++v) rotary += in->vehicle_kind[v] == FP_ROTARY;
  int* chosen = (int*)malloc(sizeof(int) * (B + 1));
  int nch = 0, heli = 0;
  for (int k = 0; k < B; ++k) {
    if (nch == V) break;
    const int bi = order[k];
    const int h = in->base_kind[bi] == FP_HELIPAD;
    if (h && heli == rotary) continue;
    chosen[nch++] = bi;
    heli += h;
  }
  int rc = FP_OK;
  if (nch < V) { rc = FP_ERR_VALIDATION; goto done; }
  {
    int* rot = (int*)malloc(sizeof(int) * (V + 1));
    int* fix = (int*)malloc(sizeof(int) * (V + 1));
    int nr = 0, nf = 0;
    for (int v = 0; v < V; ++v) {
      if (in->vehicle_kind[v] == FP_ROTARY) rot[nr++] = in->vehicle_id[v];
      else fix[nf++] = in->vehicle_id[v];
    }
    qsort(rot, (size_t)nr, sizeof(int), cmp_int);
    qsort(fix, (size_t)nf, sizeof(int), cmp_int);
    int* base_vehicle = (int*)malloc(sizeof(int) * (B + 1));
    for (int b = 0; b < B; ++b) base_vehicle[b] = -1;
    for (int v = 0; v < V; ++v) out->vehicle_base[v] = -1;
    int next_r = 0, next_f = 0;
    /* id -> index for vehicles (linear; oracle sizes are small) */
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = 0; k < nch; ++k) {
        const int bi = chosen[k];
        const int h = in->base_kind[bi] == FP_HELIPAD;
        if ((pass == 0) != h) continue;
        const int vid = pass == 0 ? rot[next_r++] : (next_r < nr ? rot[next_r++] : fix[next_f++]);
        int vi = -1;
        for (int v = 0; v < V; ++v) if (in->vehicle_id[v] == vid) { vi = v; break; }
        base_vehicle[bi] = vi;
        out->vehicle_base[vi] = bi;
      }
    }
    for (int64_t m = 0; m < M; ++m) {
      int best = -1;
      double best_cost = 0.0;
      for (int k = 0; k < nch; ++k) {
        const int bi = chosen[k];
        const int vi = base_vehicle[bi];
        if (in->rotary_only[m] && in->vehicle_kind[vi] == FP_FIXED) continue;
        const double c = cost[(int64_t)bi * M + m];
        if (best < 0 || c < best_cost || (c == best_cost && in->base_id[bi] < in->base_id[best])) {
          best = bi;
          best_cost = c;
        }
      }
      if (best < 0) { rc = FP_ERR_NO_COMPATIBLE; break; }
      out->mission_vehicle[m] = base_vehicle[best];
    }
    if (rc == FP_OK) {
      int nu = 0;
      for (int k = 0; k < B; ++k)
        if (base_vehicle[order[k]] < 0) out->unused_bases[nu++] = order[k];
      out->n_unused = nu;
    }
    free(rot);
    free(fix);
    free(base_vehicle);
  }
done:
  free(order);
  free(chosen);
  return rc;
}

/* -------------------------------------------------------------- search --- */
typedef struct { int kind, index; } pool_e;

typedef struct {
  int64_t key;     /* (kind << 40) | (id + 2^31), or -1 for an empty slot */
  int64_t expiry;
  int role;        /* 0 outer, 1 inner */
} tabu_slot;

typedef struct {
  tabu_slot* s;
  int64_t cap;
} tabu_map;

static int64_t tkey(int kind, int id) {
  return ((int64_t)kind << 40) | ((int64_t)id + 2147483648LL);
}
static tabu_slot* tabu_find(tabu_map* t, int64_t key, int create) {
  uint64_t h = (uint64_t)key * 0x9E3779B97F4A7C15ULL;
  for (int64_t k = (int64_t)(h >> 20) & (t->cap - 1);; k = (k + 1) & (t->cap - 1)) {
    if (t->s[k].key == key) return &t->s[k];
    if (t->s[k].key == -1) {
      if (!create) return NULL;
      t->s[k].key = key;
      t->s[k].expiry = 0;
      t->s[k].role = 0;
      return &t->s[k];
    }
  }
}

typedef struct {
  const fp_instance* in;
  const double* cost;
  int64_t M;
  int B, V;
  int* vehicle_base;
  int* mission_vehicle;
  int* base_vehicle;
  int* vehicle_missions;
  pool_e* pool;
  int pool_size;
  double* mission_cost;
  double total;
} state;

typedef struct {
  int kind, mission, gain, target, pool_pos, jside;
  double quick;
} cand;

static double C(const state* st, int64_t m, int b) { return st->cost[(int64_t)b * st->M + m]; }

static double resum(const state* st) {
  double s = 0.0;
  for (int64_t m = 0; m < st->M; ++m) s += st->mission_cost[m];
  return s;
}

static int eval_takeover(const state* st, int i, int j, cand* c) {
  if (i < 0 || i >= st->pool_size) return 0;
  if (st->pool[i].kind != FP_POOL_IDLE_VEHICLE) return 0;
  const int gain = st->pool[i].index;
  if (st->in->rotary_only[j] && st->in->vehicle_kind[gain] == FP_FIXED) return 0;
  c->kind = FP_MOVE_TAKEOVER;
  c->mission = j;
  c->gain = gain;
  c->target = -1;
  c->pool_pos = i;
  c->jside = st->mission_vehicle[j];
  c->quick = C(st, j, st->vehicle_base[gain]) - st->mission_cost[j];
  return 1;
}

static int eval_relocate(const state* st, int i, int j, cand* c) {
  if (i < 0 || i >= st->pool_size) return 0;
  if (st->pool[i].kind != FP_POOL_EMPTY_BASE) return 0;
  const int target = st->pool[i].index;
  const int mover = st->mission_vehicle[j];
  if (st->in->vehicle_kind[mover] == FP_FIXED && st->in->base_kind[target] == FP_HELIPAD) return 0;
  c->kind = FP_MOVE_RELOCATE;
  c->mission = j;
  c->gain = mover;
  c->target = target;
  c->pool_pos = i;
  c->jside = mover;
  double d = 0.0;
  for (int64_t m = 0; m < st->M; ++m) {
    if (st->mission_vehicle[m] != mover) continue;
    d += C(st, m, target) - st->mission_cost[m];
  }
  c->quick = d;
  return 1;
}

static int eval_reassign(const state* st, int i, int j, cand* c) {
  if (i < 0 || i >= st->M) return 0;
  const int gain = st->mission_vehicle[i];
  const int loser = st->mission_vehicle[j];
  if (gain == loser) return 0;
  if (st->in->rotary_only[j] && st->in->vehicle_kind[gain] == FP_FIXED) return 0;
  c->kind = FP_MOVE_REASSIGN;
  c->mission = j;
  c->gain = gain;
  c->target = -1;
  c->pool_pos = -1;
  c->jside = loser;
  c->quick = C(st, j, st->vehicle_base[gain]) - st->mission_cost[j];
  return 1;
}

static double candidate_total(const state* st, const cand* c) {
  double s = 0.0;
  if (c->kind == FP_MOVE_RELOCATE) {
    for (int64_t m = 0; m < st->M; ++m)
      s += st->mission_vehicle[m] == c->gain ? C(st, m, c->target) : st->mission_cost[m];
  } else {
    const double nc = C(st, c->mission, st->vehicle_base[c->gain]);
    for (int64_t m = 0; m < st->M; ++m) s += m == c->mission ? nc : st->mission_cost[m];
  }
  return s;
}

static void apply_move(state* st, const cand* c) {
  if (c->kind == FP_MOVE_TAKEOVER) {
    const int loser = st->mission_vehicle[c->mission];
    st->mission_vehicle[c->mission] = c->gain;
    st->vehicle_missions[c->gain]++;
    st->vehicle_missions[loser]--;
    st->mission_cost[c->mission] = C(st, c->mission, st->vehicle_base[c->gain]);
    if (st->vehicle_missions[loser] == 0) {
      st->pool[c->pool_pos].kind = FP_POOL_IDLE_VEHICLE;
      st->pool[c->pool_pos].index = loser;
    } else {
      memmove(st->pool + c->pool_pos, st->pool + c->pool_pos + 1,
              sizeof(pool_e) * (size_t)(st->pool_size - c->pool_pos - 1));
      st->pool_size--;
    }
  } else if (c->kind == FP_MOVE_RELOCATE) {
    const int mover = c->gain;
    const int old = st->vehicle_base[mover];
    st->base_vehicle[old] = -1;
    st->base_vehicle[c->target] = mover;
    st->vehicle_base[mover] = c->target;
    for (int64_t m = 0; m < st->M; ++m)
      if (st->mission_vehicle[m] == mover) st->mission_cost[m] = C(st, m, c->target);
    st->pool[c->pool_pos].kind = FP_POOL_EMPTY_BASE;
    st->pool[c->pool_pos].index = old;
  } else {
    const int loser = st->mission_vehicle[c->mission];
    st->mission_vehicle[c->mission] = c->gain;
    st->vehicle_missions[c->gain]++;
    st->vehicle_missions[loser]--;
    st->mission_cost[c->mission] = C(st, c->mission, st->vehicle_base[c->gain]);
    if (st->vehicle_missions[loser] == 0) {
      memmove(st->pool + 1, st->pool, sizeof(pool_e) * (size_t)st->pool_size);
      st->pool[0].kind = FP_POOL_IDLE_VEHICLE;
      st->pool[0].index = loser;
      st->pool_size++;
    }
  }
  st->total = resum(st);
}

/* Move log record, one per applied move. */
typedef struct or_move {
  int64_t tick;
  int32_t pass, kind, i, j, gain, target;
} or_move;

typedef struct {
  or_move* log;
  int64_t cap, n;
} mlog;

static int try_move(state* st, int which, int i, int j, tabu_map* tabu, int64_t tick,
                    int64_t tenure, fp_search_stats* s, mlog* log, int pass) {
  s->evaluations++;
  cand c;
  int ok = which == 0 ? eval_takeover(st, i, j, &c)
         : which == 1 ? eval_relocate(st, i, j, &c)
                      : eval_reassign(st, i, j, &c);
  if (!ok || !(c.quick < 0.0)) return 0;
  const double after = candidate_total(st, &c);
  if (!(after < st->total)) return 0;
  /* keys captured before the state mutates (proj/src/search.cpp:289-291) */
  const int okind = c.kind;
  const int oid = c.kind == FP_MOVE_RELOCATE ? st->in->base_id[c.target]
                                             : st->in->vehicle_id[c.gain];
  const int iid = st->in->vehicle_id[c.jside];
  apply_move(st, &c);
  s->applied_moves++;
  s->committed_moves++;
  if (log->log && log->n < log->cap) {
    or_move* r = &log->log[log->n];
    r->tick = tick; r->pass = pass; r->kind = c.kind; r->i = i; r->j = j;
    r->gain = c.gain; r->target = c.target;
  }
  log->n++;
  if (tabu) {
    tabu_slot* t = tabu_find(tabu, tkey(okind, oid), 1);
    t->expiry = tick + tenure;
    t->role = 0;
    if (c.kind == FP_MOVE_RELOCATE) {
      t = tabu_find(tabu, tkey(c.kind, iid), 1);
      t->expiry = tick + tenure;
      t->role = 1;
    }
  }
  return 1;
}

/* Returns: 0 = pair evaluated, 1 = inner skip, 2 = outer skip. */
static int key_state(const state* st, int i, int j, tabu_map* tabu, int64_t tick) {
  int64_t keys[3];
  int nk = 0;
  if (i >= 0 && i < st->pool_size) {
    const pool_e e = st->pool[i];
    keys[nk++] = e.kind == FP_POOL_IDLE_VEHICLE
                     ? tkey(FP_MOVE_TAKEOVER, st->in->vehicle_id[e.index])
                     : tkey(FP_MOVE_RELOCATE, st->in->base_id[e.index]);
  }
  if (i >= 0 && i < st->M)
    keys[nk++] = tkey(FP_MOVE_REASSIGN, st->in->vehicle_id[st->mission_vehicle[i]]);
  keys[nk++] = tkey(FP_MOVE_RELOCATE, st->in->vehicle_id[st->mission_vehicle[j]]);
  int blocked = 0, outer = 0;
  for (int k = 0; k < nk; ++k) {
    tabu_slot* t = tabu_find(tabu, keys[k], 0);
    if (t && tick < t->expiry) {
      blocked = 1;
      if (t->role == 0) outer = 1;
    }
  }
  return outer ? 2 : blocked;
}

/*
 * tabu_search / local_search restated. `start` is the SearchState::from
 * input (assignment + full pool, already the output of initial_pool).
 * Preconditions of SearchState::from and the tenure/mode checks are the
 * caller's (the Python wrapper mirrors them); this returns FP_OK.
 */
int or_search(const fp_instance* in, const double* cost, const fp_search_config* cfg,
              const fp_search_start* start, fp_search_result* out, or_move* log,
              int64_t log_cap, int64_t* log_n) {
  state st;
  st.in = in;
  st.cost = cost;
  st.M = in->n_missions;
  st.B = in->n_bases;
  st.V = in->n_vehicles;
  st.vehicle_base = (int*)malloc(sizeof(int) * (st.V + 1));
  st.mission_vehicle = (int*)malloc(sizeof(int) * (st.M + 1));
  st.base_vehicle = (int*)malloc(sizeof(int) * (st.B + 1));
  st.vehicle_missions = (int*)calloc((size_t)st.V + 1, sizeof(int));
  st.pool = (pool_e*)malloc(sizeof(pool_e) * (size_t)(start->pool_size + st.V + 1));
  st.mission_cost = (double*)malloc(sizeof(double) * (st.M + 1));
  for (int b = 0; b < st.B; ++b) st.base_vehicle[b] = -1;
  for (int v = 0; v < st.V; ++v) {
    st.vehicle_base[v] = start->vehicle_base[v];
    if (st.vehicle_base[v] >= 0) st.base_vehicle[st.vehicle_base[v]] = v;
  }
  for (int64_t m = 0; m < st.M; ++m) {
    st.mission_vehicle[m] = start->mission_vehicle[m];
    st.vehicle_missions[st.mission_vehicle[m]]++;
  }
  for (int64_t m = 0; m < st.M; ++m)
    st.mission_cost[m] = C(&st, m, st.vehicle_base[st.mission_vehicle[m]]);
  st.total = resum(&st);
  st.pool_size = start->pool_size;
  for (int k = 0; k < start->pool_size; ++k) {
    st.pool[k].kind = start->pool_kind[k];
    st.pool[k].index = start->pool_index[k];
  }

  tabu_map tabu_storage, *tabu = NULL;
  int64_t tenure = 0;
  if (cfg->mode == FP_MODE_TABU) {
    tenure = cfg->tabu_tenure > 0 ? cfg->tabu_tenure : 2 * st.M;
    int64_t cap = 64;
    while (cap < 4 * (st.B + 2 * st.V) + 64) cap <<= 1;
    tabu_storage.cap = cap;
    tabu_storage.s = (tabu_slot*)malloc(sizeof(tabu_slot) * (size_t)cap);
    for (int64_t k = 0; k < cap; ++k) tabu_storage.s[k].key = -1;
    tabu = &tabu_storage;
  }

  mlog lg = {log, log_cap, 0};
  or_mt64 rng;
  mt_seed(&rng, cfg->seed);
  const int n = (int)st.M;
  int* pa = (int*)malloc(sizeof(int) * (n + 1));
  int* pb = (int*)malloc(sizeof(int) * (n + 1));
  fp_search_stats s;
  memset(&s, 0, sizeof(s));
  int64_t tick = 0;
  int passes = 0;
  int keep_going = 1;
  while (keep_going) {
    random_permutation(&rng, n, pa);
    random_permutation(&rng, n, pb);
    const uint64_t applied_before = s.applied_moves;
    const uint64_t skips_before = s.tabu_skips_outer + s.tabu_skips_inner;
    for (int a = 0; a < n; ++a) {
      const int i = pa[a];
      for (int b = 0; b < n; ++b) {
        const int j = pb[b];
        if (tabu) {
          const int ks = key_state(&st, i, j, tabu, tick);
          if (ks) {
            tick++;
            if (ks == 2) { s.tabu_skips_outer++; break; }
            s.tabu_skips_inner++;
            continue;
          }
        }
        for (int which = 0; which < 3; ++which)
          try_move(&st, which, i, j, tabu, tick, tenure, &s, &lg, passes);
        if (tabu) tick++;
      }
    }
    const int improved = s.applied_moves != applied_before;
    const int blocked = s.tabu_skips_outer + s.tabu_skips_inner != skips_before;
    keep_going = tabu ? (improved || blocked) : improved;
    ++passes;
    if (cfg->max_passes >= 0 && passes >= cfg->max_passes) break;
  }
  s.passes = (uint64_t)passes;
  s.final_objective_km = st.total;
  out->stats = s;
  for (int v = 0; v < st.V; ++v) out->vehicle_base[v] = st.vehicle_base[v];
  for (int64_t m = 0; m < st.M; ++m) out->mission_vehicle[m] = st.mission_vehicle[m];
  if (log_n) *log_n = lg.n;
  free(pa);
  free(pb);
  if (tabu) free(tabu_storage.s);
  free(st.vehicle_base);
  free(st.mission_vehicle);
  free(st.base_vehicle);
  free(st.vehicle_missions);
  free(st.pool);
  free(st.mission_cost);
  return FP_OK;
}

/* Fixed mission-order objective (proj/src/model.cpp:176-192). */
double or_objective_km(int32_t M, const double* cost, const int32_t* vehicle_base,
                       const int32_t* mission_vehicle) {
  double s = 0.0;
  for (int64_t m = 0; m < M; ++m) s += cost[(int64_t)vehicle_base[mission_vehicle[m]] * M + m];
  return s;
}
