// search_kernels.cu — kernels (3)+(4): the Tabu / local-search automaton.
//
// One thread block runs one scenario's search pass (grid = scenarios). The
// block replays the reference's sequential first-improvement automaton
// exactly (proj/src/search.cpp:277-346, 401-434; SURVEY.md §8a "normative
// automaton") but finds the next EVENT data-parallel:
//
//  * Row skipping. Most rows of perm_a end at their first pair on an outer
//    tabu block (SURVEY.md §7 design notes). NT upcoming rows are tested in
//    parallel under the assumption that each earlier row took one tick; the
//    first row that is not outer-blocked at p = 0 is the next interesting
//    row, the rows before it are consumed at one tick each.
//  * Row scanning. For an interesting row, perm_b positions are scanned in
//    chunks of NT*U. Before the first event no state changes, so every pair
//    can be classified independently: outer-blocked (event: row ends),
//    inner-blocked (tick + skip), or evaluated (3 evaluations); an evaluated
//    pair is an event when one of its three moves MAY be accepted
//    (takeover/reassign: new cost < current cost; relocation: the per-vehicle
//    delta class is not certainly >= 0). A block argmin over the position
//    finds the first event; counts before it give the SearchStats increments.
//  * Event pairs are processed exactly as the reference does (takeover, then
//    relocation, then reassignment, each on the state the previous one left)
//    with the exact accept rule quick_delta < 0 && candidate_total < total.
//    The fixed-order fp64 sums are decided by a rigorous error bound; only
//    candidates inside the bound fall back to the exact sequential chains
//    (SURVEY.md §7 hard part 1).
//
// The tabu list is the expiry-stamp form (live iff tick < expiry), held in
// dense per-key arrays; the {Relocate, id} key space is shared by base and
// vehicle ids exactly like the reference's std::map<TabuKey, Entry>.

#include <cfloat>
#include <climits>

#include "common.cuh"

namespace fpk {

namespace {

constexpr int U = 4;  // positions per thread per chunk
enum : uint8_t { CLS_POS = 0, CLS_NEG = 1, CLS_ACC = 2, CLS_AMB = 3 };
constexpr double kTwoPowM52 = 2.220446049250313e-16;  // 2^-52

struct Shared {
  Counters c;                 // block copy of the counters
  // row context (written by thread 0, read by all)
  int gain_r, col_r, fixed_r;           // reassignment gainer = vehicle of mission i
  int gain_t, col_t, fixed_t;           // takeover gainer (pool[i] idle) or -1
  int rel_t, heli_t;                    // relocation target (pool[i] empty) or -1
  int lim_ro, lim_ra;                   // row keys: live-positions (outer / any)
  long long t0;                         // tick at the start of the scan segment
  int bi[8];
  double bd[4];
  int red_i[2][33];
  double red_d[3][33];
};

// Phase timing (thread 0's SM clock), accumulated into Counters::cycles.
__device__ __forceinline__ long long ph_now() { return threadIdx.x == 0 ? clock64() : 0; }
#define PH_ADD(sh, k, t0) \
  do {                    \
    if (threadIdx.x == 0) (sh).c.cycles[k] += clock64() - (t0); \
  } while (0)

__device__ __forceinline__ double cost_at(const Scenario& s, int col, int m) {
  return s.cost[(long long)col * s.M + m];
}

template <int NT>
__device__ int block_min(int v, Shared& sh) {
  v = __reduce_min_sync(0xffffffffu, v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh.red_i[0][w] = v;
  __syncthreads();
  if (w == 0) {
    int x = l < NT / 32 ? sh.red_i[0][l] : INT_MAX;
    x = __reduce_min_sync(0xffffffffu, x);
    if (l == 0) sh.red_i[0][32] = x;
  }
  __syncthreads();
  const int r = sh.red_i[0][32];
  __syncthreads();
  return r;
}

template <int NT>
__device__ void block_sum2(int& a, int& b, Shared& sh) {
  a = (int)__reduce_add_sync(0xffffffffu, (unsigned)a);
  b = (int)__reduce_add_sync(0xffffffffu, (unsigned)b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sh.red_i[0][w] = a;
    sh.red_i[1][w] = b;
  }
  __syncthreads();
  if (w == 0) {
    int x = l < NT / 32 ? sh.red_i[0][l] : 0;
    int y = l < NT / 32 ? sh.red_i[1][l] : 0;
    x = (int)__reduce_add_sync(0xffffffffu, (unsigned)x);
    y = (int)__reduce_add_sync(0xffffffffu, (unsigned)y);
    if (l == 0) {
      sh.red_i[0][32] = x;
      sh.red_i[1][32] = y;
    }
  }
  __syncthreads();
  a = sh.red_i[0][32];
  b = sh.red_i[1][32];
  __syncthreads();
}

template <int NT>
__device__ void block_sum3d(double& a, double& b, double& c, Shared& sh) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sh.red_d[0][w] = a;
    sh.red_d[1][w] = b;
    sh.red_d[2][w] = c;
  }
  __syncthreads();
  if (w == 0) {
    double x = l < NT / 32 ? sh.red_d[0][l] : 0.0;
    double y = l < NT / 32 ? sh.red_d[1][l] : 0.0;
    double z = l < NT / 32 ? sh.red_d[2][l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_down_sync(0xffffffffu, x, o);
      y += __shfl_down_sync(0xffffffffu, y, o);
      z += __shfl_down_sync(0xffffffffu, z, o);
    }
    if (l == 0) {
      sh.red_d[0][32] = x;
      sh.red_d[1][32] = y;
      sh.red_d[2][32] = z;
    }
  }
  __syncthreads();
  a = sh.red_d[0][32];
  b = sh.red_d[1][32];
  c = sh.red_d[2][32];
  __syncthreads();
}

// Rigorous bound for a single-substitution candidate (takeover/reassign):
// with S, S' the fixed-order fp64 sums before/after replacing one term by a
// smaller one, |S - X| and |S' - X'| are each <= gamma_{M-1} * X, so
// S' < S whenever the exact decrease exceeds 2 gamma_{M-1} X
// <= (M + 2) 2^-52 total_up.
__device__ __forceinline__ double single_bound(const Scenario& s, const Shared& sh) {
  return (double)(s.M + 2) * kTwoPowM52 * sh.c.total_up * 1.0001;
}

// Exact fixed-order sums S (current) and S' (mission j charged newc),
// proj/src/search.cpp:150-167 and proj/src/search_state.hpp:36-40.
// Thread 0 only.
__device__ bool exact_single_accept(const Scenario& s, int j, double newc) {
  double a = 0.0, b = 0.0;
  for (int m = 0; m < s.M; ++m) {
    const double c = s.mc[m];
    a += c;
    b += m == j ? newc : c;
  }
  return b < a;
}

// Exact relocation quick delta, proj/src/search.cpp:121-127. Thread 0.
__device__ double exact_reloc_quick(const Scenario& s, int t, int mover) {
  double d = 0.0;
  const double* col = s.cost + (long long)t * s.M;
  for (int m = 0; m < s.M; ++m)
    if (s.mv[m] == mover) d += col[m] - s.mc[m];
  return d;
}

// Exact relocation candidate_total < total. Thread 0.
__device__ bool exact_reloc_accept(const Scenario& s, int t, int mover) {
  double a = 0.0, b = 0.0;
  const double* col = s.cost + (long long)t * s.M;
  for (int m = 0; m < s.M; ++m) {
    const double c = s.mc[m];
    a += c;
    b += s.mv[m] == mover ? col[m] : c;
  }
  return b < a;
}

// Per-vehicle relocation deltas towards target base t, in any order, with
// the data needed for a rigorous sign/accept classification.
template <int NT>
__device__ void reloc_sums(const Scenario& s, int t, double* sumD, double* absD,
                           int* cnt) {
  for (int v = threadIdx.x; v < s.V; v += NT) {
    sumD[v] = 0.0;
    absD[v] = 0.0;
    cnt[v] = 0;
  }
  __syncthreads();
  const double* col = s.cost + (long long)t * s.M;
  for (int m = threadIdx.x; m < s.M; m += NT) {
    const int v = s.mv[m];
    const double d = col[m] - s.mc[m];
    atomicAdd(&sumD[v], d);
    atomicAdd(&absD[v], fabs(d));
    atomicAdd(&cnt[v], 1);
  }
  __syncthreads();
}

// Classification of one vehicle's relocation (see header comment):
// POS  quick_delta >= 0 for sure (never accepted)
// NEG  quick_delta < 0 for sure, the total comparison is not yet settled
// ACC  accepted for sure
// AMB  sign of the sequential quick_delta not settled
__device__ __forceinline__ uint8_t reloc_class(double sum, double abs, int n,
                                               double bound_total) {
  // all terms exactly zero (e.g. a base at the same location): the
  // sequential sum is exactly 0.0, never < 0
  if (n == 0 || abs == 0.0) return CLS_POS;
  const double err = (double)(n + 1) * kTwoPowM52 * abs * 1.0001;
  if (sum > err) return CLS_POS;
  if (sum < -(err + bound_total)) return CLS_ACC;
  if (sum < -err) return CLS_NEG;
  return CLS_AMB;
}

__device__ __forceinline__ bool compat_vm(bool vehicle_fixed, bool rotary_only) {
  return !(vehicle_fixed && rotary_only);
}

// ---- moves (proj/src/search.cpp:169-220) ---------------------------------
// Thread 0 only unless noted.

__device__ void set_mission(const Scenario& s, int j, int v, double c) {
  s.mv[j] = v;
  s.mc[j] = c;
  const int q = s.invb[j];
  s.mvp[q] = v;
  s.mcp[q] = c;
}

__device__ void apply_takeover(const Scenario& s, Shared& sh, int j, int gain, int pos) {
  const int loser = s.mv[j];
  set_mission(s, j, gain, cost_at(s, s.vbase[gain], j));
  s.vcount[gain] += 1;
  s.vcount[loser] -= 1;
  if (s.vcount[loser] == 0) {
    s.pkind[pos] = POOL_IDLE;
    s.pidx[pos] = loser;
  } else {
    for (int k = pos; k + 1 < sh.c.psize; ++k) {
      s.pkind[k] = s.pkind[k + 1];
      s.pidx[k] = s.pidx[k + 1];
    }
    sh.c.psize -= 1;
  }
}

__device__ void apply_reassign(const Scenario& s, Shared& sh, int j, int gain) {
  const int loser = s.mv[j];
  set_mission(s, j, gain, cost_at(s, s.vbase[gain], j));
  s.vcount[gain] += 1;
  s.vcount[loser] -= 1;
  if (s.vcount[loser] == 0) {
    for (int k = sh.c.psize; k > 0; --k) {
      s.pkind[k] = s.pkind[k - 1];
      s.pidx[k] = s.pidx[k - 1];
    }
    s.pkind[0] = POOL_IDLE;
    s.pidx[0] = loser;
    sh.c.psize += 1;
  }
}

// Block-cooperative relocation of `mover` to base t through pool slot pos.
template <int NT>
__device__ void apply_relocate(const Scenario& s, Shared& sh, int mover, int t, int pos) {
  const double* col = s.cost + (long long)t * s.M;
  for (int m = threadIdx.x; m < s.M; m += NT)
    if (s.mv[m] == mover) {
      const double c = col[m];
      s.mc[m] = c;
      s.mcp[s.invb[m]] = c;
    }
  if (threadIdx.x == 0) {
    const int old = s.vbase[mover];
    s.bveh[old] = -1;
    s.bveh[t] = mover;
    s.vbase[mover] = t;
    s.pkind[pos] = POOL_EMPTY;
    s.pidx[pos] = old;
  }
  __syncthreads();
}

// debug_check_deltas (proj/src/search.cpp:266-271): the reference recomputes
// objective_km, which throws InfeasibleError on an infeasible state
// (proj/src/model.cpp:176-181), and compares it with the running total. Our
// total is exact by construction, so the check reduces to the state's
// feasibility and its per-mission cost bookkeeping. Thread 0.
__device__ void debug_check(const Scenario& s, Shared& sh) {
  for (int v = 0; v < s.V; ++v) {
    const int b = s.vbase[v];
    if (b < 0 || (s.vfixed[v] && s.bheli[b])) { sh.c.error = 3; return; }
    for (int w = v + 1; w < s.V; ++w)
      if (s.vbase[w] == b) { sh.c.error = 3; return; }
  }
  for (int m = 0; m < s.M; ++m) {
    const int v = s.mv[m];
    if (s.ro[m] && s.vfixed[v]) { sh.c.error = 3; return; }
    if (s.mc[m] != cost_at(s, s.vbase[v], m)) { sh.c.error = 6; return; }
  }
}

__device__ void insert_outer(const Scenario& s, long long* arr, int idx, long long exp) {
  arr[idx] = exp;
}

// Processes the pair (i, j) exactly as try_move x3 (proj/src/search.cpp:277-303,
// 333-341). Block-cooperative; returns with the block synchronised.
template <int NT>
__device__ void process_pair(const Scenario& s, Shared& sh, int i, int j, bool tabu,
                             long long tenure, bool debug, double* sumD, double* absD,
                             int* cnt) {
  const long long exp = sh.c.tick + tenure;
  // ---- takeover
  if (threadIdx.x == 0) {
    sh.c.evaluations += 1;
    if (i < sh.c.psize && s.pkind[i] == POOL_IDLE) {
      const int g = s.pidx[i];
      if (compat_vm(s.vfixed[g], s.ro[j])) {
        const double newc = cost_at(s, s.vbase[g], j);
        const double mcj = s.mc[j];
        if (newc - mcj < 0.0) {
          bool acc = mcj - newc > single_bound(s, sh);
          if (!acc) {
            const long long f0 = ph_now();
            sh.c.fallbacks += 1;
            acc = exact_single_accept(s, j, newc);
            PH_ADD(sh, 4, f0);
          }
          if (acc) {
            apply_takeover(s, sh, j, g, i);
            sh.c.applied += 1;
            sh.c.pass_applied += 1;
            if (tabu) insert_outer(s, s.exp_take, g, exp);
            if (debug) debug_check(s, sh);
          }
        }
      }
    }
    // relocation preconditions (on the state the takeover left)
    sh.c.evaluations += 1;
    int t = -1, mover = -1;
    if (i < sh.c.psize && s.pkind[i] == POOL_EMPTY) {
      t = s.pidx[i];
      mover = s.mv[j];
      if (s.vfixed[mover] && s.bheli[t]) t = -1;
    }
    sh.bi[0] = t;
    sh.bi[1] = mover;
  }
  __syncthreads();
  // ---- relocation
  const int t = sh.bi[0], mover = sh.bi[1];
  if (t >= 0) {
    // sums for the mover only
    double a = 0.0, b = 0.0, c = 0.0;
    const double* col = s.cost + (long long)t * s.M;
    for (int m = threadIdx.x; m < s.M; m += NT)
      if (s.mv[m] == mover) {
        const double d = col[m] - s.mc[m];
        a += d;
        b += fabs(d);
        c += 1.0;
      }
    block_sum3d<NT>(a, b, c, sh);
    if (threadIdx.x == 0) {
      const double bt = single_bound(s, sh);
      const uint8_t cls = reloc_class(a, b, (int)c, bt);
      bool acc = cls == CLS_ACC;
      if (cls == CLS_NEG || cls == CLS_AMB) {
        const long long f0 = ph_now();
        sh.c.fallbacks += 1;
        const bool neg = cls == CLS_NEG || exact_reloc_quick(s, t, mover) < 0.0;
        acc = neg && exact_reloc_accept(s, t, mover);
        PH_ADD(sh, 4, f0);
      }
      sh.bi[2] = acc;
    }
    __syncthreads();
    if (sh.bi[2]) {
      apply_relocate<NT>(s, sh, mover, t, i);
      if (threadIdx.x == 0) {
        sh.c.applied += 1;
        sh.c.pass_applied += 1;
        if (tabu) {
          // outer {Relocate, target base id} then inner {Relocate, mover id};
          // the second insert wins when the two ids coincide.
          const int ko = s.brk[t], ki = s.vrk[mover];
          s.exp_rel[ko] = exp;
          s.role_rel[ko] = ROLE_OUTER;
          s.exp_rel[ki] = exp;
          s.role_rel[ki] = ROLE_INNER;
        }
        if (debug) debug_check(s, sh);
      }
    }
  }
  // ---- reassignment
  if (threadIdx.x == 0) {
    sh.c.evaluations += 1;
    const int g = s.mv[i], l = s.mv[j];
    if (g != l && compat_vm(s.vfixed[g], s.ro[j])) {
      const double newc = cost_at(s, s.vbase[g], j);
      const double mcj = s.mc[j];
      if (newc - mcj < 0.0) {
        bool acc = mcj - newc > single_bound(s, sh);
        if (!acc) {
          const long long f0 = ph_now();
          sh.c.fallbacks += 1;
          acc = exact_single_accept(s, j, newc);
          PH_ADD(sh, 4, f0);
        }
        if (acc) {
          apply_reassign(s, sh, j, g);
          sh.c.applied += 1;
          sh.c.pass_applied += 1;
          if (tabu) insert_outer(s, s.exp_reas, g, exp);
          if (debug) debug_check(s, sh);
        }
      }
    }
    sh.c.tick += 1;
  }
  __syncthreads();
}

// Row context after any state change (thread 0 writes, all read after sync).
template <int NT>
__device__ void make_context(const Scenario& s, Shared& sh, int i, bool tabu, int* lim_j,
                             uint8_t* outer_j, uint8_t* cls, double* sumD, double* absD,
                             int* cnt) {
  if (threadIdx.x == 0) {
    const int g = s.mv[i];
    sh.gain_r = g;
    sh.col_r = s.vbase[g];
    sh.fixed_r = s.vfixed[g];
    sh.gain_t = -1;
    sh.rel_t = -1;
    int lim_ro = 0, lim_ra = 0;
    const long long T = sh.c.tick;
    sh.t0 = T;
    if (i < sh.c.psize) {
      const int k = s.pkind[i], x = s.pidx[i];
      if (k == POOL_IDLE) {
        sh.gain_t = x;
        sh.col_t = s.vbase[x];
        sh.fixed_t = s.vfixed[x];
        if (tabu) {
          const long long e = s.exp_take[x] - T;
          const int lim = e <= 0 ? 0 : (e > s.M + 1 ? s.M + 1 : (int)e);
          lim_ro = lim;
          lim_ra = lim;
        }
      } else {
        sh.rel_t = x;
        sh.heli_t = s.bheli[x];
        if (tabu) {
          const int kk = s.brk[x];
          const long long e = s.exp_rel[kk] - T;
          const int lim = e <= 0 ? 0 : (e > s.M + 1 ? s.M + 1 : (int)e);
          if (s.role_rel[kk] == ROLE_OUTER) lim_ro = lim;
          lim_ra = lim;
        }
      }
    }
    if (tabu) {
      const long long e = s.exp_reas[g] - T;
      const int lim = e <= 0 ? 0 : (e > s.M + 1 ? s.M + 1 : (int)e);
      lim_ro = max(lim_ro, lim);
      lim_ra = max(lim_ra, lim);
    }
    sh.lim_ro = lim_ro;
    sh.lim_ra = lim_ra;
  }
  __syncthreads();
  if (tabu) {
    const long long T = sh.t0;
    for (int v = threadIdx.x; v < s.V; v += NT) {
      const int k = s.vrk[v];
      const long long e = s.exp_rel[k] - T;
      lim_j[v] = e <= 0 ? 0 : (e > s.M + 1 ? s.M + 1 : (int)e);
      outer_j[v] = s.role_rel[k] == ROLE_OUTER;
    }
  }
  const int t = sh.rel_t;
  if (t >= 0) {
    const long long r0 = ph_now();
    reloc_sums<NT>(s, t, sumD, absD, cnt);
    const double bt = single_bound(s, sh);
    for (int v = threadIdx.x; v < s.V; v += NT)
      cls[v] = (s.vfixed[v] && sh.heli_t) ? CLS_POS : reloc_class(sumD[v], absD[v], cnt[v], bt);
    PH_ADD(sh, 5, r0);
  }
  __syncthreads();
}

// One outer-index row, proj/src/search.cpp:307-346.
template <int NT>
__device__ void run_row(const Scenario& s, Shared& sh, int i, const int32_t* __restrict__ pb,
                        bool tabu, long long tenure, bool debug, int* lim_j, uint8_t* outer_j,
                        uint8_t* cls, double* sumD, double* absD, int* cnt) {
  const int M = s.M;
  int p = 0;
  while (p < M) {
    const long long c0 = ph_now();
    make_context<NT>(s, sh, i, tabu, lim_j, outer_j, cls, sumD, absD, cnt);
    PH_ADD(sh, 1, c0);
    const long long c1 = ph_now();
    const int p_seg = p;
    const int gain_r = sh.gain_r, col_r = sh.col_r, fixed_r = sh.fixed_r;
    const int gain_t = sh.gain_t, col_t = sh.col_t, fixed_t = sh.fixed_t;
    const int rel_t = sh.rel_t;
    const int lim_ro = sh.lim_ro, lim_ra = sh.lim_ra;
    int ev = INT_MAX;
    while (p < M) {
      // classify U positions per thread; bit k of `inner`/`unb` marks status
      unsigned inner = 0, unb = 0;
      int first = INT_MAX;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int q = p + k * NT + threadIdx.x;
        if (q >= M) break;
        const int v = s.mvp[q];
        if (tabu) {
          const int off = q - p_seg;
          const int lj = lim_j[v];
          const bool oj = outer_j[v];
          if (off < lim_ro || (off < lj && oj)) {
            first = min(first, q);
            break;
          }
          if (off < lim_ra || off < lj) {
            inner |= 1u << k;
            continue;
          }
        }
        const int j = pb[q];
        const double mcj = s.mcp[q];
        const bool roj = s.rop[q];
        bool e = false;
        if (gain_t >= 0 && compat_vm(fixed_t, roj)) e |= cost_at(s, col_t, j) < mcj;
        if (rel_t >= 0) e |= cls[v] != CLS_POS;
        if (v != gain_r && compat_vm(fixed_r, roj)) e |= cost_at(s, col_r, j) < mcj;
        if (e) {
          first = min(first, q);
          break;
        }
        unb |= 1u << k;
      }
      ev = block_min<NT>(first, sh);
      int n_in = 0, n_unb = 0;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int q = p + k * NT + threadIdx.x;
        if (q >= ev || q >= M) break;
        n_in += (inner >> k) & 1u;
        n_unb += (unb >> k) & 1u;
      }
      block_sum2<NT>(n_in, n_unb, sh);
      const int chunk_end = min(p + NT * U, M);
      const int stop = min(ev, chunk_end);
      if (threadIdx.x == 0) {
        sh.c.skips_inner += (unsigned long long)n_in;
        sh.c.evaluations += 3ull * (unsigned long long)n_unb;
        if (tabu) sh.c.tick += stop - p;
        if (n_in > 0) sh.c.pass_skipped = 1;
      }
      __syncthreads();
      p = stop;
      if (ev != INT_MAX) break;
    }
    PH_ADD(sh, 2, c1);
    if (ev == INT_MAX) return;  // row exhausted perm_b
    // event at position p
    bool outer_ev = false;
    if (tabu) {
      const int v = s.mvp[p];
      const int off = p - p_seg;
      outer_ev = off < lim_ro || (off < lim_j[v] && outer_j[v]);
    }
    if (outer_ev) {
      if (threadIdx.x == 0) {
        sh.c.skips_outer += 1;
        sh.c.tick += 1;
        sh.c.pass_skipped = 1;
      }
      __syncthreads();
      return;
    }
    const long long c2 = ph_now();
    process_pair<NT>(s, sh, i, pb[p], tabu, tenure, debug, sumD, absD, cnt);
    PH_ADD(sh, 3, c2);
    __syncthreads();
    if (sh.c.error) return;
    p += 1;
  }
}

}  // namespace

// Rebuild the perm_b-ordered mirrors for a new pass.
__global__ void mirror_kernel(Scenario* scs, const int32_t* __restrict__ active,
                              const int32_t* __restrict__ pb) {
  if (!active[blockIdx.y]) return;
  const Scenario s = scs[blockIdx.y];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < s.M; q += gridDim.x * blockDim.x) {
    const int j = pb[q];
    s.mvp[q] = s.mv[j];
    s.mcp[q] = s.mc[j];
    s.rop[q] = s.ro[j];
    s.invb[j] = q;
  }
}

// One pass over perm_a for every active scenario (blockIdx.x = scenario).
template <int NT>
__global__ void __launch_bounds__(NT, NT == 1024 ? 1 : 4)
    pass_kernel(Scenario* scs, const int32_t* __restrict__ active, const int32_t* __restrict__ pa,
                const int32_t* __restrict__ pb, int tabu_i, long long tenure, int debug_i) {
  if (!active[blockIdx.x]) return;
  const Scenario s = scs[blockIdx.x];
  const bool tabu = tabu_i != 0, debug = debug_i != 0;
  __shared__ Shared sh;
  extern __shared__ __align__(16) unsigned char dyn[];
  double* sumD = reinterpret_cast<double*>(dyn);
  double* absD = sumD + s.V;
  int* lim_j = reinterpret_cast<int*>(absD + s.V);
  int* cnt = lim_j + s.V;
  uint8_t* outer_j = reinterpret_cast<uint8_t*>(cnt + s.V);
  uint8_t* cls = outer_j + s.V;
  if (threadIdx.x == 0) {
    sh.c = *s.ctr;
    sh.c.pass_applied = 0;
    sh.c.pass_skipped = 0;
  }
  __syncthreads();
  const int M = s.M;
  int r = 0;
  while (r < M && !sh.c.error) {
    const long long b0 = ph_now();
    if (tabu) {
      // rows r .. r+NT-1: outer-blocked at p = 0 if every earlier one was?
      const int d = threadIdx.x, row = r + d;
      int cand = INT_MAX;
      if (row < M) {
        const int i = pa[row];
        const long long T = sh.c.tick + d;
        bool outer = T < s.exp_reas[s.mv[i]];
        if (i < sh.c.psize) {
          const int x = s.pidx[i];
          if (s.pkind[i] == POOL_IDLE) {
            outer |= T < s.exp_take[x];
          } else {
            const int k = s.brk[x];
            outer |= T < s.exp_rel[k] && s.role_rel[k] == ROLE_OUTER;
          }
        }
        const int k = s.vrk[s.mvp[0]];
        outer |= T < s.exp_rel[k] && s.role_rel[k] == ROLE_OUTER;
        if (!outer) cand = d;
      }
      const int found = block_min<NT>(cand, sh);
      const int nskip = found == INT_MAX ? min(NT, M - r) : found;
      if (threadIdx.x == 0 && nskip > 0) {
        sh.c.tick += nskip;
        sh.c.skips_outer += (unsigned long long)nskip;
        sh.c.pass_skipped = 1;
      }
      __syncthreads();
      r += nskip;
      PH_ADD(sh, 0, b0);
      if (found == INT_MAX) continue;
    }
    run_row<NT>(s, sh, pa[r], pb, tabu, tenure, debug, lim_j, outer_j, cls, sumD, absD, cnt);
    __syncthreads();
    r += 1;
  }
  if (threadIdx.x == 0) *s.ctr = sh.c;
}

// Search start: per-mission costs, per-vehicle counts and the exact initial
// total (SearchState::from, proj/src/search.cpp:41-48). One block per
// scenario; the fixed-order total is one sequential chain (thread 0).
__global__ void init_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.x];
  for (int m = threadIdx.x; m < s.M; m += blockDim.x)
    s.mc[m] = cost_at(s, s.vbase[s.mv[m]], m);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int m = 0; m < s.M; ++m) t += s.mc[m];
    s.ctr->total_up = t;
    s.ctr->final_total = t;
  }
}

// Exact fixed-order final total (st.total after the last move).
__global__ void final_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.x];
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int m = 0; m < s.M; ++m) t += s.mc[m];
    s.ctr->final_total = t;
  }
}

size_t pass_dyn_smem(int V) { return (size_t)V * (8 + 8 + 4 + 4 + 1 + 1) + 16; }

cudaError_t launch_pass(Scenario* d_scs, const int32_t* d_active, int n_scn, const int32_t* d_pa,
                        const int32_t* d_pb, int M, bool tabu, long long tenure, bool debug, int V,
                        cudaStream_t stream, int threads) {
  const size_t smem = pass_dyn_smem(V);
  dim3 mg((M + 255) / 256 < 64 ? (M + 255) / 256 : 64, n_scn);
  if (M > 0) mirror_kernel<<<mg, 256, 0, stream>>>(d_scs, d_active, d_pb);
  if (threads == 1024) {
    cudaFuncSetAttribute(pass_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_kernel<1024><<<n_scn, 1024, smem, stream>>>(d_scs, d_active, d_pa, d_pb, tabu, tenure,
                                                    debug);
  } else {
    cudaFuncSetAttribute(pass_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_kernel<256><<<n_scn, 256, smem, stream>>>(d_scs, d_active, d_pa, d_pb, tabu, tenure,
                                                  debug);
  }
  return cudaGetLastError();
}

cudaError_t launch_init(Scenario* d_scs, int n_scn, cudaStream_t stream) {
  init_kernel<<<n_scn, 256, 0, stream>>>(d_scs);
  return cudaGetLastError();
}

cudaError_t launch_final(Scenario* d_scs, int n_scn, cudaStream_t stream) {
  final_kernel<<<n_scn, 32, 0, stream>>>(d_scs);
  return cudaGetLastError();
}

}  // namespace fpk
