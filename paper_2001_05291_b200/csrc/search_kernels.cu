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
//    delta class is not certainly >= 0). All loads of a chunk are issued
//    before any is consumed; one ballot-based block reduction yields the
//    first event and the SearchStats increments before it.
//  * Event pairs are processed exactly as the reference does (takeover, then
//    relocation, then reassignment, each on the state the previous one left)
//    with the exact accept rule quick_delta < 0 && candidate_total < total.
//    The fixed-order fp64 sums are decided by a rigorous error bound; only
//    candidates inside the bound fall back to the exact sequential chains
//    (SURVEY.md §7 hard part 1).
//
// The tabu list is the expiry-stamp form (live iff tick < expiry), held in
// dense per-key arrays; the {Relocate, id} key space is shared by base and
// vehicle ids exactly like the reference's std::map<TabuKey, Entry>. The
// per-vehicle / per-key state lives in shared memory for the whole pass.

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#ifdef FP_ROW_TRACE
#include <cstdio>
#endif

namespace fpk {

namespace {

enum : uint8_t { CLS_POS = 0, CLS_NEG = 1, CLS_ACC = 2, CLS_AMB = 3 };
constexpr double kTwoPowM52 = 2.220446049250313e-16;  // 2^-52
constexpr unsigned FULL = 0xffffffffu;

struct Shared {
  Counters c;                 // block copy of the counters
  int bi[8];
  int ev;                               // scan step result broadcast
  int nj;                               // live j-keys in sm.jl_*
  int nrl;                              // vehicles whose relocation class is not POS (sm.rlist)
  long long jexp_max;                   // latest expiry of any vehicle's {Relocate, id} key
  long long jkey_ver;                   // {Relocate, id} inserts so far in this launch
  long long jl_ver;                     // jkey_ver when the j-key list was built (-1: never)
  int tmp;
  double bd0;
  double xs;                            // exact chain: partial sum so far ...
  int xk;                               // ... after this many terms
  unsigned hk;                          // helper jobs posted in this launch
  unsigned hdone;                       // helper completions expected so far
  unsigned lt, lsync, ldone0;           // substitution log: published, applied, base
  int hp2_from;                         // hP2 holds the last candidate chain from this chunk (-1: none)
  int reassigned;                       // process_pair applied a reassignment (its last move kind)
  long long red_l[33];
  int red_i[2][33];
  int red2[2][32][2];                   // row-run minima, double-buffered
  double red_d[3][33];
};

// Dynamic shared memory carve-up (see pass_smem_bytes()).
struct Smem {
  int* lim_j;          // [V] positions from the segment start a j-key stays live
  uint8_t* outer_j;    // [V] that key's role is Outer
  uint8_t* cls;        // [V] relocation class towards the row's empty base
  double* acc_sum;     // [NW*V] warp-private relocation partial sums
  double* acc_abs;     // [NW*V]
  double* stage;       // [NW*32]
  int* wsum;           // [NW*3] per-warp scan summaries
  int* xidx;           // [2*NT] mission-index buffer for exact relocation deltas
  int* xlist;          // position buffer for relocation bitset updates (global scratch)
  int xlist_cap;
  int* impc;           // [V] set bits of imp[g] (0 = no reassign/takeover to g improves)
  int* rlist;          // [V] vehicles whose relocation to the row's empty base may improve
  int* jl_v;           // [V] vehicles whose {Relocate, id} j-key is live
  long long* jl_exp;   // [V] its expiry stamp (live iff tick < stamp)
  uint8_t* jl_outer;   // [V] its role is Outer
  const int32_t* pb;   // perm_b
  int* paw;            // [2*NT] window of perm_a (row runs)
  int helpers;         // helper blocks sharing relocations (0 = none)
  unsigned epoch;      // launch number (helper job tags)
  int32_t* gvbase;     // global vbase (helpers read the mover's new base)
  int32_t* gmv;        // global mv / mvp when the block works on shared-memory
  int32_t* gmvp;       //   copies (written through), else null
};

// Phase timing (thread 0's SM clock), accumulated into Counters::cycles.
// Phase clocks (SearchStats::phase_cycles): probe builds only
// (FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS): thread 0's clock reads and
// shared-memory accumulations cost the automaton ~5% (c2 to quiescence 112
// -> 107 ms, the c5 share 193 -> 182 ms without them).
#ifndef FP_PHASE_CLOCKS
__device__ __forceinline__ long long ph_now() { return 0; }
#define PH_ADD(sh, k, t0) \
  do {                    \
  } while (0)
#else
__device__ __forceinline__ long long ph_now() { return threadIdx.x == 0 ? clock64() : 0; }
#define PH_ADD(sh, k, t0)                                        \
  do {                                                           \
    if (threadIdx.x == 0) (sh).c.cycles[k] += clock64() - (t0); \
  } while (0)
#endif

__device__ __forceinline__ double cost_at(const Scenario& s, int col, int m) {
  return s.cost[(long long)col * s.M + m];
}

// The same entry for accesses that run over bases with the mission fixed
// (one mission's costs at every base are contiguous in the row-major copy).
__device__ __forceinline__ double cost_mb(const Scenario& s, int m, int b) {
  return s.costT ? s.costT[(long long)m * s.B + b] : s.cost[(long long)b * s.M + m];
}

__device__ __forceinline__ int clamp_lim(long long e, int M) {
  return e <= 0 ? 0 : (e > M + 1 ? M + 1 : (int)e);
}

template <int NT>
__device__ int block_min(int v, Shared& sh) {
  v = __reduce_min_sync(FULL, v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh.red_i[0][w] = v;
  __syncthreads();
  if (w == 0) {
    int x = l < NT / 32 ? sh.red_i[0][l] : INT_MAX;
    x = __reduce_min_sync(FULL, x);
    if (l == 0) sh.red_i[0][32] = x;
  }
  __syncthreads();
  const int r = sh.red_i[0][32];
  __syncthreads();
  return r;
}

// Rigorous bound for a single-substitution candidate (takeover/reassign):
// with S, S' the fixed-order fp64 sums before/after replacing one term by a
// smaller one, |S - X| and |S' - X'| are each <= gamma_{M-1} * X, so
// S' < S whenever the exact decrease exceeds 2 gamma_{M-1} X
// <= (M + 2) 2^-52 total_up.
__device__ __forceinline__ double single_bound(const Scenario& s, const Shared& sh) {
  if (sh.c.force_exact & 1) return INFINITY;
  return (double)(s.M + 2) * kTwoPowM52 * sh.c.total_up * 1.0001;
}

// ---- exact fixed-order fp64 sums, block-parallel -------------------------
//
// The reference decides candidate_total < total with two sequential fp64
// sums over the M mission costs (proj/src/search.cpp:150-167, search_state.hpp
// :36-40). exact_chain reproduces such a sum bit for bit with the whole
// block: while the running sum S stays in one binade [2^e, 2^(e+1)) every
// partial sum is a multiple of u = 2^(e-52), so fl(S + c) = S + u*rn(c/u)
// unless c/u is an exact tie (then round-to-even depends on S). A chunk of
// terms is therefore an int64 prefix scan of rn(c/u); the step that leaves
// the binade is done with one true fp64 add from the exact integer-form
// partial sum, and a chunk holding a tie before its crossing is stepped
// sequentially up to the tie. All terms are >= 0 (distances), so S is
// monotone and crosses each binade once.
//   kind 0: c_k = mc[k]                      (the current total)
//   kind 1: c_k = (k == j ? newc : mc[k])    (takeover / reassignment)
//   kind 2: c_k = (mv[k] == mover ? col[k] : mc[k])   (relocation)
__device__ __forceinline__ double chain_term(const Scenario& s, int kind, int k, int j, double newc,
                                             int mover, const double* col) {
  if (kind == 1) return k == j ? newc : s.mc[k];
  if (kind == 2) return s.mv[k] == mover ? col[k] : s.mc[k];
  return s.mc[k];
}

// ---- helper blocks (large single scenarios) --------------------------------
//
// A relocation touches O(M) state: the mover's missions get new costs, the
// mover's imp row is rebuilt, the bits of its positions change in every
// other row, and the vacated base needs a fresh relocation row. For large
// scenarios that work is split over helper blocks that wait in the same
// launch; the master block shifts the other table rows meanwhile. The
// handshake is a release/acquire pair at gpu scope on HelperCtl::seq and
// HelperCtl::done; all spins are bounded (a hang guard that reports an error).

constexpr long long kSpinLimit = 1ll << 35;  // ~17 s of SM clock

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Master, thread 0: publish a job (the block's earlier writes are ordered
// before it by the caller's barrier).
__device__ void post_job(const Scenario& s, Shared& sh, const Smem& sm, int kind, int x, int t,
                         int b_old) {
  HelperCtl* hc = s.hc;
  hc->kind = kind;
  hc->x = x;
  hc->t = t;
  hc->b_old = b_old;
  sh.hk += 1;
  __threadfence();
  st_release_u64(&hc->seq, ((unsigned long long)sm.epoch << 32) | sh.hk);
}

// Master, block-wide: wait until every helper finished the last job.
template <int NT>
__device__ void wait_helpers(const Scenario& s, Shared& sh, const Smem& sm) {
  if (threadIdx.x == 0) {
    sh.hdone += (unsigned)sm.helpers;
    const long long t0 = clock64();
    while ((int)(ld_acquire_u32(&s.hc->done) - sh.hdone) < 0) {
      if (clock64() - t0 > kSpinLimit) {
        sh.c.error = 8;  // FP_ERR_CUDA: helper blocks stopped answering
        break;
      }
      __nanosleep(32);
    }
    sh.c.cycles[14] += (unsigned long long)(clock64() - t0);
  }
  __syncthreads();
}

template <int NT>
__device__ long long block_inclusive_scan(long long x, Shared& sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  long long incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(FULL, incl, o);
    if (l >= o) incl += y;
  }
  if (l == 31) sh.red_l[w] = incl;
  __syncthreads();
  long long before = 0;
  for (int k = 0; k < w; ++k) before += sh.red_l[k];
  __syncthreads();
  return before + incl;
}

// Master, thread 0: publish a substitution record for the helpers' table
// patches (back-pressure: a full log is drained first).
__device__ void log_wait(const Scenario& s, Shared& sh, const Smem& sm) {
  const long long t0 = clock64();
  const unsigned want = (unsigned)sm.helpers * sh.lt;
  while ((int)(ld_acquire_u32(&s.hc->log_done) - sh.ldone0 - want) < 0) {
    if (clock64() - t0 > kSpinLimit) {
      sh.c.error = 8;
      break;
    }
    __nanosleep(32);
  }
  sh.c.cycles[14] += (unsigned long long)(clock64() - t0);
  sh.lsync = sh.lt;
}

__device__ void log_append(const Scenario& s, Shared& sh, const Smem& sm, int j, int loser,
                           int gain, int nl, int ng, double mc_old, double mc_new) {
  if (sh.lt - sh.lsync >= (unsigned)kLogCap) log_wait(s, sh, sm);
  SubRec r;
  r.j = j;
  r.loser = loser;
  r.gain = gain;
  r.nl = nl;
  r.ng = ng;
  r.pad = 0;
  r.mc_old = mc_old;
  r.mc_new = mc_new;
  s.hlog[sh.lt % kLogCap] = r;
  sh.lt += 1;
  __threadfence();
  st_release_u64(&s.hc->log_tail, ((unsigned long long)sm.epoch << 32) | sh.lt);
}

// Block-wide: every published record applied to the table (before any read
// of rA / rE / rU / rcnt in helper mode). Uniform: sh.lt / sh.lsync are only
// written by thread 0 before a barrier.
template <int NT, bool HELP>
__device__ void table_sync(const Scenario& s, Shared& sh, const Smem& sm) {
  if (!HELP || sm.helpers == 0 || sh.lt == sh.lsync) return;
  if (threadIdx.x == 0) log_wait(s, sh, sm);
  __syncthreads();
}

// rn(x / u) for u = 2^(e-52) (an exact power-of-two scaling), with the
// tie flag; x >= 4e15 u certainly leaves the binade in one step.
__device__ __forceinline__ long long chain_round(double x, double inv_u, bool& tie) {
  const double y = x * inv_u;
  tie = false;
  if (y >= 4.0e15) return 1ll << 53;
  const double f = floor(y);
  const double fr = y - f;
  tie = fr == 0.5;
  return (long long)f + (fr >= 0.5 ? 1 : 0);
}

// Advances the exact chain held in (sh.xk, sh.xs) to term kend. Each step
// covers 32*UE consecutive terms per warp (coalesced); the first EVENT of a
// step -- the term whose addition leaves the binade, or a rounding tie
// (round-half-even then depends on the running sum) -- is found by the warp
// whose range holds it with one lane scan per 32 terms; the sum before it
// is exact in integer form and the event itself is one true fp64 add. Every
// kChainSub-aligned boundary a step passes gets its binade recorded in
// s.hec (the prediction exact_chain_helped hands to its helpers).
template <int NT>
__device__ void chain_steps(const Scenario& s, Shared& sh, int kind, int j, double newc,
                            int mover, const double* col, int kend) {
  constexpr int NW = NT / 32;
  constexpr int UE = 32;
  constexpr long long LIM = 1ll << 53;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    double S = sh.xs;
    int k = sh.xk;
    while (k < kend && !(S >= 0x1p-900)) {  // leading zeros / tiny values: plain adds
      S += chain_term(s, kind, k, j, newc, mover, col);
      ++k;
    }
    sh.xs = S;
    sh.xk = k;
  }
  __syncthreads();
  while (true) {
    const int k0 = sh.xk;
    const double S0 = sh.xs;
    if (k0 >= kend) break;
    const int e = ilogb(S0);
    const double u = ldexp(1.0, e - 52), inv_u = ldexp(1.0, 52 - e);
    const long long N0 = (long long)(S0 * inv_u);
    // warp range [wb, wb + 32*nq): lane l holds terms wb + 32q + l; the
    // warp's integer total is order-free. Short ranges are spread over all
    // warps (one load round instead of nq).
    const int per = min(32 * UE, (((kend - k0 + NW - 1) / NW) + 31) & ~31);
    const int nq = per >> 5;
    const int wb = k0 + w * per;
    long long local = 0;
    int first_tie = INT_MAX;
#pragma unroll 8
    for (int q = 0; q < nq; ++q) {
      const int k = wb + q * 32 + l;
      if (k < kend) {
        bool tie = false;
        local += chain_round(chain_term(s, kind, k, j, newc, mover, col), inv_u, tie);
        if (tie) first_tie = min(first_tie, k);
      }
    }
    // saturate: only reaching LIM matters. A lane holds up to 32 terms of
    // <= LIM each (2^58); clamping it before the warp sum keeps that sum
    // <= 2^58 too -- unclamped, 1024 saturated terms (a chain whose first
    // term is small against the next 1024) sum to 2^63 and wrap negative,
    // hiding the binade crossing
#ifndef FP_CHAIN_UNCLAMPED  // (probe builds: the round-2 bug, to show the test catches it)
    local = min(local, LIM);
#endif
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(FULL, local, o);
    local = min(local, LIM);
    first_tie = __reduce_min_sync(FULL, first_tie);
    if (l == 0) sh.red_l[w] = local;
    __syncthreads();
    long long run = N0, total = 0;
    for (int k = 0; k < NW; ++k) {
      const long long v = sh.red_l[k];
      if (k < w) run += v;
      total += v;
    }
    int first_ev = INT_MAX;
    long long before_ev = 0;
    if (run + local >= LIM || first_tie != INT_MAX) {
      for (int q = 0; q < nq; ++q) {
        const int k = wb + q * 32 + l;
        long long r = 0;
        bool tq = false;
        if (k < kend) r = chain_round(chain_term(s, kind, k, j, newc, mover, col), inv_u, tq);
        long long incl = r;
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(FULL, incl, o);
          if (l >= o) incl += y;
        }
        const unsigned hit = __ballot_sync(FULL, k < kend && (tq || run + incl >= LIM));
        if (hit) {
          const int f = __ffs(hit) - 1;
          const long long excl = __shfl_sync(FULL, incl - r, f);
          first_ev = wb + q * 32 + f;
          before_ev = run + excl;
          break;
        }
        run += __shfl_sync(FULL, incl, 31);
      }
    }
    const int ev = block_min<NT>(first_ev, sh);
    // aligned boundaries in [k0, lim] have their running sum in binade e
    const int lim = ev == INT_MAX ? min(kend, k0 + per * NW) : ev;
    {
      // (hec has one entry per chunk start: c < ceil(M / kChainSub); a chain
      // ending exactly on a chunk boundary must not record the next one)
      const int c = (k0 + kChainSub - 1) / kChainSub + threadIdx.x;
      if ((long long)c * kChainSub <= lim && c < (s.M + kChainSub - 1) / kChainSub) s.hec[c] = e;
    }
    if (ev == INT_MAX) {
      if (threadIdx.x == 0) {
        sh.xs = (double)(N0 + total) * u;
        sh.xk = min(kend, k0 + per * NW);
      }
    } else if (first_ev == ev && l == 0) {
      // exact partial sum before the event, then the event's true fp64 add
      const double prev = (double)before_ev * u;
      sh.xs = prev + chain_term(s, kind, ev, j, newc, mover, col);
      sh.xk = ev + 1;
    }
    __syncthreads();
  }
}

template <int NT>
__device__ double exact_chain(const Scenario& s, Shared& sh, int kind, int j, double newc,
                              int mover, const double* col) {
  // The head of a chain from zero crosses a binade every time the running
  // sum doubles (~log2(k) events in its first k terms, each a block step):
  // its first kChainSeqHead terms are summed by one thread with plain fp64
  // adds in order -- the reference's own loop, exact by definition -- and
  // the block steps take over once the running sum is large.
  // (warp 0: coalesced loads of 32 terms, the next 32 in flight while every
  // lane adds the current ones in order from shuffles)
  constexpr int kChainSeqHead = 1024;
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    const int kh = min(s.M, kChainSeqHead);
    double S = 0.0;
    double nxt = l < kh ? chain_term(s, kind, l, j, newc, mover, col) : 0.0;
    for (int k0 = 0; k0 < kh; k0 += 32) {
      const double cur = nxt;
      const int kk = k0 + 32 + l;
      if (kk < kh) nxt = chain_term(s, kind, kk, j, newc, mover, col);
      const int n = min(32, kh - k0);
      for (int q = 0; q < n; ++q) S += __shfl_sync(FULL, cur, q);
    }
    if (l == 0) {
      sh.xs = S;
      sh.xk = kh;
    }
  }
  __syncthreads();
  chain_steps<NT>(s, sh, kind, j, newc, mover, col, s.M);
  const double r = sh.xs;
  __syncthreads();
  return r;
}

// Helper share of an exact chain: for chunks part, part + parts, ... the
// sum of rn(term / u) in the binade the latest chain recorded for the
// chunk's start, with that binade in hue -- or kNoBinade when the chunk
// holds a rounding tie or a term that leaves the binade by itself (or no
// binade is known).
template <int NT>
__device__ void helper_chain(const Scenario& s, Shared& sh, int kind, int j, double newc,
                             int mover, int t, int part, int parts) {
  constexpr int NW = NT / 32;
  constexpr long long LIM = 1ll << 53;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int M = s.M;
  const double* col = t >= 0 ? s.cost + (long long)t * M : nullptr;
  const int nsub = (M + kChainSub - 1) / kChainSub;
  const int c0 = __ldcg(&s.hc->cstart);
  for (int c = c0 + part; c < nsub; c += parts) {
    const int e = __ldcg(&s.hec[c]);
    if (e == kNoBinade) {
      if (threadIdx.x == 0) s.hue[c] = kNoBinade;
      continue;
    }
    const double inv_u = ldexp(1.0, 52 - e);
    long long local = 0;
    bool flag = false;
#pragma unroll 4
    for (int q = 0; q < kChainSub / NT; ++q) {
      const int k = c * kChainSub + q * NT + threadIdx.x;
      if (k < M) {
        bool tie = false;
        const long long r = chain_round(chain_term(s, kind, k, j, newc, mover, col), inv_u, tie);
        flag |= tie || r >= LIM;
        local = min(local + r, LIM);
      }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(FULL, local, o);
    local = min(local, LIM);
    const bool wf = __any_sync(FULL, flag);
    if (l == 0) {
      sh.red_l[w] = local;
      sh.red_i[1][w] = wf;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long tot = 0;
      int f = 0;
      for (int k = 0; k < NW; ++k) {
        tot = min(tot + sh.red_l[k], LIM);
        f |= sh.red_i[1][k];
      }
      s.hrs[c] = tot;
      s.hue[c] = f ? kNoBinade : e;
    }
    __syncthreads();
  }
}

// Exact chain with the helper blocks: the helpers sum every chunk's rounded
// terms in its predicted binade (the binade recorded by the latest chain:
// one move changes the sums too little to move most chunk boundaries across
// a binade); the master then walks the chunks, consuming NT chunks per block
// scan while the prediction holds (same binade, no tie, no crossing inside),
// and runs chain_steps on every other chunk. Block-wide.
template <int NT>
__device__ double exact_chain_helped(const Scenario& s, Shared& sh, const Smem& sm, int kind,
                                     int j, double newc, int mover, int t, int c0, int rec) {
  double* const hp = rec == 1 ? s.hP : s.hP2;
  const bool record = rec != 0;
  constexpr long long LIM = 1ll << 53;
  const int M = s.M;
  const double* col = t >= 0 ? s.cost + (long long)t * M : nullptr;
  __syncthreads();
  if (threadIdx.x == 0) {
    HelperCtl* hc = s.hc;
    hc->ckind = kind;
    hc->cj = j;
    hc->cmover = mover;
    hc->ct = t;
    hc->cnewc = newc;
    hc->cstart = c0;
    post_job(s, sh, sm, HJOB_CHAIN, 0, 0, 0);
  }
  wait_helpers<NT>(s, sh, sm);
  // the chain is the current state's up to chunk c0: start from its
  // recorded exact running sum there
  if (threadIdx.x == 0) {
    sh.xs = c0 > 0 ? s.hP[c0] : 0.0;
    sh.xk = c0 * kChainSub;
  }
  __syncthreads();
  const int nsub = (M + kChainSub - 1) / kChainSub;
  while (true) {
    const int k = sh.xk;
    const double S = sh.xs;
    if (k >= M || sh.c.error) break;
    if (k % kChainSub != 0 || !(S >= 0x1p-900)) {
      if (record && k % kChainSub == 0 && threadIdx.x == 0) hp[k / kChainSub] = S;
      chain_steps<NT>(s, sh, kind, j, newc, mover, col, min(M, (k / kChainSub + 1) * kChainSub));
      continue;
    }
    const int e = ilogb(S);
    const double u = ldexp(1.0, e - 52), inv_u = ldexp(1.0, 52 - e);
    const long long N = (long long)(S * inv_u);
    const int c = k / kChainSub;
    const int cc = c + threadIdx.x;
    // hue, not hec: the walk itself re-records hec as it goes
    const bool ok = cc < nsub && __ldcg(&s.hue[cc]) == e;
    const long long v = ok ? __ldcg(&s.hrs[cc]) : 0;
    const long long incl = block_inclusive_scan<NT>(v, sh);
    const bool good = ok && N + incl < LIM;
    const int bad = block_min<NT>(good ? INT_MAX : (int)threadIdx.x, sh);
    const int nok = bad == INT_MAX ? NT : bad;
    if (record && (int)threadIdx.x < nok) hp[cc] = (double)(N + incl - v) * u;
    if (nok > 0 && (int)threadIdx.x == nok - 1) {
      sh.xs = (double)(N + incl) * u;
      sh.xk = min(M, (c + nok) * kChainSub);
    }
    __syncthreads();
    if (nok < NT && sh.xk < M) {
      if (record && threadIdx.x == 0) hp[sh.xk / kChainSub] = sh.xs;
      chain_steps<NT>(s, sh, kind, j, newc, mover, col, min(M, (c + nok + 1) * kChainSub));
    }
  }
  if (record && threadIdx.x == 0 && !sh.c.error) {
    hp[nsub] = sh.xs;  // (a start at c0 = nsub returns the total itself)
    if (rec == 1) sh.c.hp_valid = nsub;
    else sh.hp2_from = c0;
  }
  const double r = sh.xs;
  __syncthreads();
  return r;
}

// Exact chain, with the helpers when there are any and M is large.
// c0: first chunk whose terms may differ from the current state's (the chain
// resumes from hP[c0] when helper-assisted); rec: 1 = the chain is the
// current state's (kind 0) and refreshes hP, 2 = a candidate's, recorded in
// hP2 (adopt_candidate_sums makes it current when the move is applied).
template <int NT, bool HELP>
__device__ double exact_chain_any(const Scenario& s, Shared& sh, const Smem& sm, int kind, int j,
                                  double newc, int mover, int t, int c0, int rec) {
  if (threadIdx.x == 0 && rec == 2) sh.hp2_from = -1;
  if (HELP && sm.helpers > 0 && s.M >= 8 * kChainSub && sh.c.chain_mode == 0)
    return exact_chain_helped<NT>(s, sh, sm, kind, j, newc, mover, t, min(c0, sh.c.hp_valid),
                                  rec);
  return exact_chain<NT>(s, sh, kind, j, newc, mover,
                         t >= 0 ? s.cost + (long long)t * s.M : nullptr);
}

// The applied move is the last candidate chain's state: its recorded running
// sums become the current ones. Block-wide.
template <int NT>
__device__ void adopt_candidate_sums(const Scenario& s, Shared& sh) {
  const int from = sh.hp2_from;
  if (from < 0) return;
  const int nsub = (s.M + kChainSub - 1) / kChainSub;
  for (int c = from + threadIdx.x; c <= nsub; c += NT) s.hP[c] = s.hP2[c];
  __syncthreads();
  if (threadIdx.x == 0) {
    sh.c.hp_valid = nsub;
    sh.hp2_from = -1;
  }
  __syncthreads();
}

// Exact current total, cached per applied-move count.
template <int NT, bool HELP>
__device__ double exact_total(const Scenario& s, Shared& sh, const Smem& sm) {
  if (sh.c.total_ver == (long long)sh.c.applied) return sh.c.total_exact;
  const long long e0 = ph_now();
  const double t = exact_chain_any<NT, HELP>(s, sh, sm, 0, -1, 0.0, -1, -1, INT_MAX, 1);
  PH_ADD(sh, 9, e0);
  if (threadIdx.x == 0) {
    sh.c.total_exact = t;
    sh.c.total_ver = (long long)sh.c.applied;
  }
  __syncthreads();
  return t;
}

// Exact relocation quick delta (proj/src/search.cpp:121-127): the mover's
// terms in ascending mission order. The block compacts the mover's mission
// indices (order preserving) into `idx`, thread 0 adds them in order.
template <int NT>
__device__ double exact_reloc_quick(const Scenario& s, Shared& sh, const double* col, int mover,
                                    int* idx, int cap) {
  constexpr int NW = NT / 32;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sh.tmp = 0;
    sh.xs = 0.0;
  }
  __syncthreads();
  for (int base = 0; base < s.M; base += NT) {
    const int m = base + threadIdx.x;
    const bool mine = m < s.M && s.mv[m] == mover;
    const unsigned b = __ballot_sync(FULL, mine);
    if (l == 0) sh.red_i[0][w] = __popc(b);
    __syncthreads();
    int off = sh.tmp;
    for (int k = 0; k < w; ++k) off += sh.red_i[0][k];
    if (mine) {
      const int pos = off + __popc(b & ((1u << l) - 1u));
      if (pos < cap) idx[pos] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int k = 0; k < NW; ++k) t += sh.red_i[0][k];
      // flush a full buffer into the running sum, in order
      int n = sh.tmp + t;
      if (n > cap - NT) {
        double d = sh.xs;
        for (int k = 0; k < n && k < cap; ++k) d += col[idx[k]] - s.mc[idx[k]];
        sh.xs = d;
        n = 0;
      }
      sh.tmp = n;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double d = sh.xs;
    for (int k = 0; k < sh.tmp; ++k) d += col[idx[k]] - s.mc[idx[k]];
    sh.xs = d;
  }
  __syncthreads();
  const double r = sh.xs;
  __syncthreads();
  return r;
}


__device__ __forceinline__ bool compat_vm(bool vehicle_fixed, bool rotary_only) {
  return !(vehicle_fixed && rotary_only);
}

// bits [0, n) of a word, n clamped to [0, 32]
__device__ __forceinline__ uint32_t prefix_bits(long long n) {
  return n <= 0 ? 0u : (n >= 32 ? FULL : ((1u << n) - 1u));
}

// imp[g] bit of position q (mission j): reassigning / taking it over to g
// lowers its cost (proj/src/search.cpp:82-101, 131-148 preconditions + sign).
__device__ __forceinline__ bool imp_bit(const Scenario& s, int g, int q, int j) {
  return s.mvp[q] != g && compat_vm(s.vfixed[g], s.rop[q]) &&
         cost_mb(s, j, s.vbase[g]) < s.mcp[q];
}

__device__ __forceinline__ void put_bit(uint32_t* w, uint32_t bit, bool on) {
  *w = on ? (*w | bit) : (*w & ~bit);
}

// After mission j at position q moved from `loser` to `gain` (new cost in
// mcp[q]): refresh bit q of every imp row, move its mem bit. Block-wide.
template <int NT>
__device__ void table_after_substitution(const Scenario& s, const Shared& sh, int j, int loser,
                                         int gain, double mc_old, double mc_new, int nl, int ng);
__device__ __forceinline__ void subst_entry(const Scenario& s, int t, double c, double Al,
                                            double El, double Ul, double Ag, double Eg, double Ug,
                                            int loser, int gain, bool fl, bool fg, double mc_old,
                                            double mc_new, int nl, int ng, double bt);
__device__ __forceinline__ long long tix(const Scenario& s, int t, int v);

// After mission j at position q moved from `loser` (cost mc_old, nl missions)
// to `gain` (new cost in mcp[q], ng missions): refresh bit q of every imp
// row, move its mem bit, and patch the relocation-delta table, in one
// block-wide phase with a single barrier.
template <int NT, bool HELP>
__device__ void bits_after_substitution(const Scenario& s, Shared& sh, const Smem& sm, int q,
                                        int j, int loser, int gain, double mc_old, double mc_new,
                                        int nl, int ng) {
  const int wd = q >> 5;
  const uint32_t bit = 1u << (q & 31);
  // One base per thread (B <= NT, no helpers): the table entries this
  // thread patches are loaded before the imp-row gathers, so both sets of
  // loads are in flight together.
  // (with helper blocks the patches of a large table go to them as a log;
  // a table of at most NT bases is patched here either way: one pass of
  // thread-per-base patches beats a wait for the log at the next row)
  const bool logged = HELP && sm.helpers > 0 && s.B > NT;
  const bool pre = !logged && s.B <= NT;
  const int t = threadIdx.x;
  const bool live = pre && t < s.B && s.bveh[t] < 0;
  double pc = 0.0, pAl = 0.0, pEl = 0.0, pUl = 0.0, pAg = 0.0, pEg = 0.0, pUg = 0.0;
  if (live) {
    pc = cost_mb(s, j, t);
    const long long kl = tix(s, t, loser), kg = tix(s, t, gain);
    pAl = s.rA[kl];
    pEl = s.rE[kl];
    pUl = s.rU[kl];
    pAg = s.rA[kg];
    pEg = s.rE[kg];
    pUg = s.rU[kg];
  }
  // The membership move and the helpers' patch record depend on nothing the
  // vehicle loop computes: two threads of the last warps (no vehicle of
  // theirs when V <= NT - 64) issue them first, so their global
  // read-modify-writes and the record's release overlap the loop's gathers.
  const long long tp0 = ph_now();
  if (threadIdx.x == NT - 1 && loser != gain) {
    s.mem[(long long)loser * s.nwd + wd] &= ~bit;
    s.mem[(long long)gain * s.nwd + wd] |= bit;
  }
  if (logged && threadIdx.x == NT - 33) log_append(s, sh, sm, j, loser, gain, nl, ng, mc_old, mc_new);
  // the first vehicle block's gathers are issued before this thread's table
  // patch, whose arithmetic then overlaps their latency
  uint32_t w_first = 0u;
  double c_first = 0.0;
  if (threadIdx.x < s.V) {
    w_first = s.imp[(long long)threadIdx.x * s.nwd + wd];
    c_first = cost_mb(s, j, s.vbase[threadIdx.x]);
  }
  if (live)
    subst_entry(s, t, pc, pAl, pEl, pUl, pAg, pEg, pUg, loser, gain, s.vfixed[loser],
                s.vfixed[gain], mc_old, mc_new, nl, ng, single_bound(s, sh));
  for (int g0 = 0; g0 < s.V; g0 += NT) {
    const int g = g0 + threadIdx.x;
    bool now = false;
    if (g < s.V) {
      uint32_t* wp = s.imp + (long long)g * s.nwd + wd;
      const uint32_t wv = g0 == 0 ? w_first : *wp;
      const double cg = g0 == 0 ? c_first : cost_mb(s, j, s.vbase[g]);
      const bool was = (wv & bit) != 0u;
      // imp_bit on the post-move state, from the move itself (thread 0 may
      // still be writing mvp[q] / mcp[q]: no barrier after the apply)
      now = gain != g && compat_vm(s.vfixed[g], s.rop[q]) && cg < mc_new;
      *wp = now ? (wv | bit) : (wv & ~bit);
      sm.impc[g] += (int)now - (int)was;
    }
    // the mission's natural-order row
    const unsigned row = __ballot_sync(FULL, now);
    if ((threadIdx.x & 31) == 0 && g < s.V) s.impT[(long long)j * s.nvw + (g >> 5)] = row;
  }
  if (logged || pre) {
  } else {
    table_after_substitution<NT>(s, sh, j, loser, gain, mc_old, mc_new, nl, ng);
  }
  PH_ADD(sh, 10, tp0);
  __syncthreads();
}

// After vehicle x moved to a new base (its missions' costs already updated):
// (1) its own imp row in full (warp per word, lane per position, 4 words in
// flight per warp); (2) the bits of the positions it serves in every other
// row: the positions are compacted from mem[x] into `list`, then the block
// runs over the flattened (position, vehicle) pairs with independent gathers
// and sets / clears bits with word atomics. Block-wide.
template <int NT>
__device__ void bits_after_relocation(const Scenario& s, Shared& sh, const Smem& sm, int x,
                                      int* list, int cap) {
  constexpr int NW = NT / 32;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nwd = s.nwd, M = s.M, V = s.V;
  const double* colx = s.cost + (long long)s.vbase[x] * M;
  const bool fx = s.vfixed[x];
  if (threadIdx.x == 0) sh.tmp = 0;
  __syncthreads();
  int cnt = 0;
  for (int wd0 = w * 8; wd0 < nwd; wd0 += NW * 8) {
    bool b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = (wd0 + u) * 32 + l;
      b[u] = false;
      if (wd0 + u < nwd && q < M)
        b[u] = s.mvp[q] != x && compat_vm(fx, s.rop[q]) && colx[sm.pb[q]] < s.mcp[q];
    }
    // bit x of the natural-order rows, where it changed
    const uint32_t xb = 1u << (x & 31);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = (wd0 + u) * 32 + l;
      if (wd0 + u < nwd && q < M) {
        const bool was = (s.imp[(long long)x * nwd + wd0 + u] >> l) & 1u;
        if (b[u] != was) {
          uint32_t* tw = s.impT + (long long)sm.pb[q] * s.nvw + (x >> 5);
          if (b[u]) atomicOr(tw, xb); else atomicAnd(tw, ~xb);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned m = __ballot_sync(FULL, b[u]);
      if (l == 0 && wd0 + u < nwd) {
        s.imp[(long long)x * nwd + wd0 + u] = m;
        cnt += __popc(m);
      }
    }
  }
  if (l == 0) atomicAdd(&sh.tmp, cnt);
  // compact the positions x serves (order irrelevant)
  if (threadIdx.x == 0) sh.bi[7] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    sm.impc[x] = sh.tmp;
  }
  for (int wd = threadIdx.x; wd < nwd; wd += NT) {
    uint32_t mx = s.mem[(long long)x * nwd + wd];
    if (mx) {
      const int at = atomicAdd(&sh.bi[7], __popc(mx));
      for (int k = at; mx; mx &= mx - 1, ++k)
        if (k < cap) list[k] = wd * 32 + __ffs(mx) - 1;
    }
  }
  __syncthreads();
  const int n = min(sh.bi[7], cap);
#ifdef FP_RELOC_PROBE
  const long long p0 = ph_now();
#endif
  // PP positions per warp at a time, lanes over vehicles: all the round's
  // gathers (PP positions x GU groups of 32 vehicles) are independent and in
  // flight together; bits of one position live in different words (rows),
  // and positions sharing a word use word atomics
  constexpr int PP = 4, GU = 2;
  for (int k0 = w * PP; k0 < n; k0 += NW * PP) {
    int qa[PP], ja[PP];
    double ma[PP];
    bool ra[PP];
#pragma unroll
    for (int a = 0; a < PP; ++a) {
      const int k = k0 + a;
      qa[a] = k < n ? list[k] : -1;
    }
#pragma unroll
    for (int a = 0; a < PP; ++a) {
      const int q = qa[a] < 0 ? 0 : qa[a];
      ja[a] = sm.pb[q];
      ma[a] = s.mcp[q];
      ra[a] = s.rop[q];
    }
    for (int g0 = 0; g0 < V; g0 += 32 * GU) {
      bool on[PP][GU];
#pragma unroll
      for (int a = 0; a < PP; ++a)
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int g = g0 + u * 32 + l;
          on[a][u] = qa[a] >= 0 && g < V && g != x && compat_vm(s.vfixed[g], ra[a]) &&
                     cost_mb(s, ja[a], s.vbase[g]) < ma[a];
        }
#pragma unroll
      for (int a = 0; a < PP; ++a) {
        if (qa[a] < 0) continue;  // warp-uniform
        const int wd = qa[a] >> 5;
        const uint32_t bit = 1u << (qa[a] & 31);
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const unsigned row = __ballot_sync(FULL, on[a][u]);
          if (l == 0 && g0 + u * 32 < V) s.impT[(long long)ja[a] * s.nvw + (g0 >> 5) + u] = row;
          const int g = g0 + u * 32 + l;
          if (g >= V || g == x) continue;
          uint32_t* wp = s.imp + (long long)g * nwd + wd;
          const uint32_t old = on[a][u] ? atomicOr(wp, bit) : atomicAnd(wp, ~bit);
          if (((old & bit) != 0u) != on[a][u]) atomicAdd(&sm.impc[g], on[a][u] ? 1 : -1);
        }
      }
    }
  }
  __syncthreads();
#ifdef FP_RELOC_PROBE
  PH_ADD(sh, 14, p0);
#endif
  if (sh.bi[7] > cap) {
    // more positions than the buffer holds: finish them one word at a time
    for (int wd = threadIdx.x; wd < nwd; wd += NT) {
      uint32_t mx = s.mem[(long long)x * nwd + wd];
      while (mx) {
        const int bn = __ffs(mx) - 1;
        mx &= mx - 1;
        const int q = wd * 32 + bn;
        const int j = sm.pb[q];
        uint32_t row = 0;
        for (int g = 0; g < V; ++g) {
          bool now = false;
          if (g != x) {
            uint32_t* wp = s.imp + (long long)g * nwd + wd;
            const bool was = (*wp & (1u << bn)) != 0u;
            now = compat_vm(s.vfixed[g], s.rop[q]) && cost_mb(s, j, s.vbase[g]) < s.mcp[q];
            put_bit(wp, 1u << bn, now);
            if (now != was) atomicAdd(&sm.impc[g], now ? 1 : -1);
          }
          row |= (uint32_t)now << (g & 31);
          if ((g & 31) == 31 || g == V - 1) {
            s.impT[(long long)j * s.nvw + (g >> 5)] = row;
            row = 0;
          }
        }
      }
    }
    __syncthreads();
  }
}

// ---- relocation-delta table ------------------------------------------------
//
// eval_relocate's quick delta (proj/src/search.cpp:121-127) depends only on
// (target base t, mover v): D(t, v) = fixed-order fp64 sum over v's missions
// of fl(cost(m, t) - mc[m]). The table keeps, per empty base t and vehicle v,
// an any-order value rA with |rA - X| <= rE around the exact real sum X and an
// upper bound rU >= sum |cost - mc|; then |D - rA| <= rE + (n + 2) 2^-52 rU
// (n = v's mission count), which classifies the relocation rigorously. Rows
// are built once by a sweep (table_rows_kernel), patched O(P) per
// reassignment / takeover (one term leaves the loser's sum, one enters the
// gainer's) and shifted per relocation (a relocation of x to t changes every
// D(t', x) by -D(t, x)); the vacated base gets a fresh row. Rounding of every
// patch is added to rE, so classes stay rigorous; a row whose bounds got too
// loose to classify (AMB) is rebuilt exactly.

// Entry (t, v) of rA/rE/rU: vehicle-major, so one vehicle's entries over
// consecutive bases are contiguous (coalesced patches after a move).
__device__ __forceinline__ long long tix(const Scenario& s, int t, int v) {
  return (long long)v * s.B + t;
}

// Class of one (t, v) entry from its values (n = v's mission count).
__device__ __forceinline__ bool table_unsettled(double A, double E0, double U, int n, double bt) {
  if (n == 0 || U == 0.0) return false;  // no terms, or every term exactly zero
  const double E = E0 + (double)(n + 2) * kTwoPowM52 * U * 1.0001;
  return !(A - E > 0.0);
  (void)bt;
}

__device__ __forceinline__ uint8_t table_class_n(const Scenario& s, const Shared& sh, int t, int v,
                                                 int n) {
  if (s.vfixed[v] && s.bheli[t]) return CLS_POS;
  const long long k = tix(s, t, v);
  const double U = s.rU[k];
  if (n == 0 || U == 0.0) return CLS_POS;  // no terms, or every term exactly zero
  const double A = s.rA[k];
  const double E = s.rE[k] + (double)(n + 2) * kTwoPowM52 * U * 1.0001;
  if (A - E > 0.0) return CLS_POS;
  if (sh.c.force_exact & 2) return CLS_AMB;
  if (A + E + single_bound(s, sh) < 0.0) return CLS_ACC;
  if (A + E < 0.0) return CLS_NEG;
  return CLS_AMB;
}

__device__ __forceinline__ uint8_t table_class(const Scenario& s, const Shared& sh, int t, int v) {
  return table_class_n(s, sh, t, v, s.vcount[v]);
}

// Fresh row t from one streaming pass over the missions (warp-private
// accumulators; lanes of a warp holding the same vehicle are grouped with
// __match_any_sync so no fp64 shared atomics are needed). Block-wide; writes
// rA/rE/rU and rcnt[t].
template <int NT>
__device__ void table_row_fresh(const Scenario& s, Shared& sh, double* acc_sum, double* acc_abs,
                                double* stage, int t) {
  constexpr int NW = NT / 32;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int V = s.V;
  double* as = acc_sum + (long long)w * V;
  double* aa = acc_abs + (long long)w * V;
  for (int v = l; v < V; v += 32) {
    as[v] = 0.0;
    aa[v] = 0.0;
  }
  double* st = stage + w * 32;
  __syncwarp();
  const double* col = s.cost + (long long)t * s.M;
  constexpr int UR = 8;  // independent 32-mission groups in flight per warp
  for (int base = w * 32; base < s.M; base += UR * NT) {
    int vv[UR];
    double dd[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int m = base + u * NT + l;
      vv[u] = -1;
      dd[u] = 0.0;
      if (m < s.M) {
        vv[u] = s.mv[m];
        dd[u] = col[m] - s.mc[m];
      }
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int v = vv[u];
      const unsigned peers = __match_any_sync(FULL, v);
      st[l] = dd[u];
      __syncwarp();
      if (v >= 0 && l == __ffs(peers) - 1) {
        double sum = 0.0, abs = 0.0;
        for (unsigned b = peers; b; b &= b - 1) {
          const double x = st[__ffs(b) - 1];
          sum += x;
          abs += fabs(x);
        }
        as[v] += sum;
        aa[v] += abs;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sh.tmp = 0;
  __syncthreads();
  int cnt = 0;
  for (int v = threadIdx.x; v < V; v += NT) {
    double sum = 0.0, abs = 0.0;
    for (int k = 0; k < NW; ++k) {
      sum += acc_sum[(long long)k * V + v];
      abs += acc_abs[(long long)k * V + v];
    }
    const int n = s.vcount[v];
    const long long k = tix(s, t, v);
    const double U = abs * (1.0 + (double)(n + 2) * kTwoPowM52);
    s.rA[k] = sum;
    s.rU[k] = U;
    s.rE[k] = (double)(n + 2) * kTwoPowM52 * U;
    cnt += table_class(s, sh, t, v) != CLS_POS;
  }
  if (cnt) atomicAdd(&sh.tmp, cnt);
  __syncthreads();
  if (threadIdx.x == 0) s.rcnt[t] = sh.tmp;
  __syncthreads();
}

// Relocation classes of every vehicle towards empty base t into sm.cls; a
// row with an unsettled class is rebuilt exactly first.
template <int NT, bool HELP>
__device__ void relocation_classes(const Scenario& s, Shared& sh, const Smem& sm, int t) {
  table_sync<NT, HELP>(s, sh, sm);
  int amb = 0;
  for (int v = threadIdx.x; v < s.V; v += NT) {
    const uint8_t c = table_class(s, sh, t, v);
    sm.cls[v] = c;
    amb |= c == CLS_AMB;
  }
  amb = __syncthreads_or(amb);
  if (amb) {
    const long long r0 = ph_now();
    if (threadIdx.x == 0) sh.c.counts[3] += 1;
    table_row_fresh<NT>(s, sh, sm.acc_sum, sm.acc_abs, sm.stage, t);
    for (int v = threadIdx.x; v < s.V; v += NT) sm.cls[v] = table_class(s, sh, t, v);
    __syncthreads();
    PH_ADD(sh, 5, r0);
  }
}


// After mission j moved from `loser` (cost mc_old, nl missions before) to
// `gain` (cost mc_new, ng missions before): patch every empty base's row and
// its count of unsettled classes. Block-wide (thread per base: the loser's
// and the gainer's entries of consecutive bases are contiguous); each entry
// is loaded once and patched in registers. Rows of empty bases outside the
// pool are kept current too (harmless; they are rebuilt fresh or patched
// the same way when they enter it).
// Entry pair (t, loser), (t, gain) of one empty base, values already loaded.
__device__ __forceinline__ void subst_entry(const Scenario& s, int t, double c, double Al,
                                            double El, double Ul, double Ag, double Eg, double Ug,
                                            int loser, int gain, bool fl, bool fg, double mc_old,
                                            double mc_new, int nl, int ng, double bt) {
  const bool heli = s.bheli[t];
  const long long kl = tix(s, t, loser), kg = tix(s, t, gain);
  int delta = 0;
  if (!(fl && heli)) delta -= table_unsettled(Al, El, Ul, nl, bt);
  if (!(fg && heli)) delta -= table_unsettled(Ag, Eg, Ug, ng, bt);
  const double dl = c - mc_old, dg = c - mc_new;
  Al -= dl;
  El += 2.0 * kTwoPowM52 * (fabs(dl) + fabs(Al));
  Ul = fmax(0.0, Ul - fabs(dl)) + 2.0 * kTwoPowM52 * Ul;
  Ag += dg;
  Eg += 2.0 * kTwoPowM52 * (fabs(dg) + fabs(Ag));
  Ug = (Ug + fabs(dg)) * (1.0 + 2.0 * kTwoPowM52);
  if (!(fl && heli)) delta += table_unsettled(Al, El, Ul, nl - 1, bt);
  if (!(fg && heli)) delta += table_unsettled(Ag, Eg, Ug, ng + 1, bt);
  s.rA[kl] = Al;
  s.rE[kl] = El;
  s.rU[kl] = Ul;
  s.rA[kg] = Ag;
  s.rE[kg] = Eg;
  s.rU[kg] = Ug;
  if (delta) s.rcnt[t] += delta;
}

template <int NT>
__device__ void table_after_substitution(const Scenario& s, const Shared& sh, int j, int loser,
                                         int gain, double mc_old, double mc_new, int nl, int ng) {
  const double bt = single_bound(s, sh);
  const bool fl = s.vfixed[loser], fg = s.vfixed[gain];
  for (int t = threadIdx.x; t < s.B; t += NT) {
    if (s.bveh[t] >= 0) continue;
    const double c = cost_mb(s, j, t);
    const long long kl = tix(s, t, loser), kg = tix(s, t, gain);
    subst_entry(s, t, c, s.rA[kl], s.rE[kl], s.rU[kl], s.rA[kg], s.rE[kg], s.rU[kg], loser, gain,
                fl, fg, mc_old, mc_new, nl, ng, bt);
  }
}

// After vehicle x moved from b_old to t (pool slot now lists b_old): every
// other empty row shifts by -D(t, x); the vacated base gets a fresh row.
template <int NT>
__device__ void table_after_relocation(const Scenario& s, Shared& sh, const Smem& sm, int x, int t,
                                       int b_old) {
  const long long kt = tix(s, t, x);
  const double At = s.rA[kt], Et = s.rE[kt], Ut = s.rU[kt];
  for (int t2 = threadIdx.x; t2 < s.B; t2 += NT) {
    if (s.bveh[t2] >= 0 || t2 == b_old) continue;
    const long long k2 = tix(s, t2, x);
    const int before = table_class(s, sh, t2, x) != CLS_POS;
    const double A = s.rA[k2] - At;
    s.rA[k2] = A;
    s.rE[k2] += Et + 2.0 * kTwoPowM52 * (fabs(At) + fabs(A));
    s.rU[k2] = (s.rU[k2] + Ut) * (1.0 + 2.0 * kTwoPowM52);
    s.rcnt[t2] += (int)(table_class(s, sh, t2, x) != CLS_POS) - before;
  }
  __syncthreads();
#ifdef FP_RELOC_PROBE
  const long long f0 = ph_now();
#endif
  table_row_fresh<NT>(s, sh, sm.acc_sum, sm.acc_abs, sm.stage, b_old);
#ifdef FP_RELOC_PROBE
  PH_ADD(sh, 9, f0);
#endif
}


// Helper share `part` of `parts` of the relocation of x from b_old to t:
//  A. missions [m0, m1): x's missions take their cost at t (mc, mcp); the bit
//     of their position in every other vehicle's imp row is recomputed; every
//     mission's term cost(m, b_old) - mc[m] is summed per vehicle into
//     hsum/habs (the vacated base's fresh relocation row, any-order sums
//     with the same rigorous bounds as table_row_fresh);
//  B. words [w0, w1) of x's own imp row.
template <int NT>
__device__ void helper_relocate(const Scenario& s, const Smem& sm, const int32_t* __restrict__ pb,
                                int x, int t, int b_old, int part, int parts) {
  constexpr int NW = NT / 32;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int V = s.V, M = s.M, nwd = s.nwd;
  int* dlt = sm.lim_j;  // [V] this block's imp-row popcount deltas
  double* as = sm.acc_sum + (long long)w * V;
  double* aa = sm.acc_abs + (long long)w * V;
  double* st = sm.stage + w * 32;
  int* list = sm.xidx;  // [2*NT]
  int* cnt = sm.wsum;
  int my_min = INT_MAX;  // smallest mission index of the mover seen by this thread
  for (int v = l; v < V; v += 32) {
    as[v] = 0.0;
    aa[v] = 0.0;
  }
  for (int v = threadIdx.x; v < V; v += NT) dlt[v] = 0;
  if (threadIdx.x == 0) *cnt = 0;
  __syncthreads();
  const double* colt = s.cost + (long long)t * M;
  const double* colo = s.cost + (long long)b_old * M;
  const int chunk = (int)((((long long)M + parts - 1) / parts + 31) & ~31ll);
  const int m0 = (int)min((long long)M, (long long)part * chunk);
  const int m1 = min(M, m0 + chunk);
  for (int base = m0; base < m1; base += NT) {
    const int m = base + threadIdx.x;
    int v = -1;
    double term = 0.0;
    if (m < m1) {
      v = s.mv[m];
      double c = s.mc[m];
      if (v == x) {
        c = colt[m];
        s.mc[m] = c;
        s.mcp[s.invb[m]] = c;
        list[atomicAdd(cnt, 1)] = m;
        my_min = min(my_min, m);
      }
      term = colo[m] - c;
    }
    const unsigned peers = __match_any_sync(FULL, v);
    st[l] = term;
    __syncwarp();
    if (v >= 0 && l == __ffs(peers) - 1) {
      double sum = 0.0, abs = 0.0;
      for (unsigned b = peers; b; b &= b - 1) {
        const double y = st[__ffs(b) - 1];
        sum += y;
        abs += fabs(y);
      }
      as[v] += sum;
      aa[v] += abs;
    }
    __syncwarp();
    __syncthreads();
    // warp per listed mission, lanes over the other vehicles
    const int n = *cnt;
    for (int k = w; k < n; k += NW) {
      const int mm = list[k];
      const int q = s.invb[mm];
      const double mcq = colt[mm];
      const bool ro = s.ro[mm];
      const uint32_t bit = 1u << (q & 31);
      const int wd = q >> 5;
      for (int g0 = 0; g0 < V; g0 += 32 * 4) {
        bool on[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int g = g0 + u * 32 + l;
          on[u] = g < V && g != x && compat_vm(s.vfixed[g], ro) && cost_mb(s, mm, s.vbase[g]) < mcq;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned row = __ballot_sync(FULL, on[u]);
          if (l == 0 && g0 + u * 32 < V) s.impT[(long long)mm * s.nvw + (g0 >> 5) + u] = row;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int g = g0 + u * 32 + l;
          if (g >= V || g == x) continue;
          uint32_t* wp = s.imp + (long long)g * nwd + wd;
          const uint32_t old = on[u] ? atomicOr(wp, bit) : atomicAnd(wp, ~bit);
          if (((old & bit) != 0u) != on[u]) atomicAdd(&dlt[g], on[u] ? 1 : -1);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) *cnt = 0;
  }
  // B. x's own row
  const bool fx = s.vfixed[x];
  const int wchunk = (nwd + parts - 1) / parts;
  const int w0 = (int)min((long long)nwd, (long long)part * wchunk);
  const int w1 = min(nwd, w0 + wchunk);
  int cb = 0;
  for (int wd0 = w0 + w * 4; wd0 < w1; wd0 += NW * 4) {
    bool b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = (wd0 + u) * 32 + l;
      b[u] = false;
      if (wd0 + u < w1 && q < M)
        b[u] = s.mvp[q] != x && compat_vm(fx, s.rop[q]) && colt[pb[q]] < s.mcp[q];
    }
    const uint32_t xb = 1u << (x & 31);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = (wd0 + u) * 32 + l;
      if (wd0 + u < w1 && q < M) {
        const bool was = (s.imp[(long long)x * nwd + wd0 + u] >> l) & 1u;
        if (b[u] != was) {
          uint32_t* tw = s.impT + (long long)pb[q] * s.nvw + (x >> 5);
          if (b[u]) atomicOr(tw, xb); else atomicAnd(tw, ~xb);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned mk = __ballot_sync(FULL, b[u]);
      if (l == 0 && wd0 + u < w1) {
        s.imp[(long long)x * nwd + wd0 + u] = mk;
        cb += __popc(mk);
      }
    }
  }
  if (l == 0 && cb) atomicAdd(&s.hc->impc_x, cb);
  my_min = __reduce_min_sync(FULL, my_min);
  if (l == 0 && my_min != INT_MAX) atomicMin(&s.hc->minm, my_min);
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += NT) {
    double sum = 0.0, abs = 0.0;
    for (int k = 0; k < NW; ++k) {
      sum += sm.acc_sum[(long long)k * V + v];
      abs += sm.acc_abs[(long long)k * V + v];
    }
    if (abs != 0.0) {
      atomicAdd(&s.hsum[v], sum);
      atomicAdd(&s.habs[v], abs);
    }
    if (dlt[v]) atomicAdd(&s.hdelta[v], dlt[v]);
  }
}

// Helper share of substitution records [from, to): the bases of slice `part`
// (thread per base; records in order, each entry patched as in
// table_after_substitution). Rows of occupied bases are patched too -- they
// are never read, and a base that empties gets a fresh row.
template <int NT>
__device__ void helper_log(const Scenario& s, unsigned from, unsigned to, int part, int parts) {
  const int per = (s.B + parts - 1) / parts;
  const int t0 = part * per, t1 = min(s.B, t0 + per);
  for (int t = t0 + threadIdx.x; t < t1; t += NT) {
    const bool heli = s.bheli[t];
    for (unsigned r = from; r < to; ++r) {
      const SubRec& rec = s.hlog[r % kLogCap];
      const int j = __ldcg(&rec.j), loser = __ldcg(&rec.loser), gain = __ldcg(&rec.gain);
      const int nl = __ldcg(&rec.nl), ng = __ldcg(&rec.ng);
      const double mc_old = __ldcg(&rec.mc_old), mc_new = __ldcg(&rec.mc_new);
      const bool fl = s.vfixed[loser], fg = s.vfixed[gain];
      const double c = cost_mb(s, j, t);
      const long long kl = tix(s, t, loser), kg = tix(s, t, gain);
      double Al = s.rA[kl], El = s.rE[kl], Ul = s.rU[kl];
      double Ag = s.rA[kg], Eg = s.rE[kg], Ug = s.rU[kg];
      int delta = 0;
      if (!(fl && heli)) delta -= table_unsettled(Al, El, Ul, nl, 0.0);
      if (!(fg && heli)) delta -= table_unsettled(Ag, Eg, Ug, ng, 0.0);
      const double dl = c - mc_old, dg = c - mc_new;
      Al -= dl;
      El += 2.0 * kTwoPowM52 * (fabs(dl) + fabs(Al));
      Ul = fmax(0.0, Ul - fabs(dl)) + 2.0 * kTwoPowM52 * Ul;
      Ag += dg;
      Eg += 2.0 * kTwoPowM52 * (fabs(dg) + fabs(Ag));
      Ug = (Ug + fabs(dg)) * (1.0 + 2.0 * kTwoPowM52);
      if (!(fl && heli)) delta += table_unsettled(Al, El, Ul, nl - 1, 0.0);
      if (!(fg && heli)) delta += table_unsettled(Ag, Eg, Ug, ng + 1, 0.0);
      s.rA[kl] = Al;
      s.rE[kl] = El;
      s.rU[kl] = Ul;
      s.rA[kg] = Ag;
      s.rE[kg] = Eg;
      s.rU[kg] = Ug;
      if (delta) s.rcnt[t] += delta;
    }
  }
}

// Helper block main loop: wait for a job of this launch (or new substitution
// records), do its share, count done; return on QUIT (or on the hang guard).
template <int NT>
__device__ void helper_loop(const Scenario& s, Shared& sh, const Smem& sm, const int32_t* pb,
                            int part, int parts) {
  unsigned seen = 0, applied = 0;
  while (true) {
    if (threadIdx.x == 0) {
      const long long t0 = clock64();
      int kind = -1;
      while (true) {
        const unsigned long long lt = ld_acquire_u64(&s.hc->log_tail);
        if ((unsigned)(lt >> 32) == sm.epoch && (unsigned)lt > applied) {
          kind = HJOB_LOG;
          sh.bi[1] = (int)(unsigned)lt;
          break;
        }
        const unsigned long long v = ld_acquire_u64(&s.hc->seq);
        if ((unsigned)(v >> 32) == sm.epoch && (unsigned)v > seen) {
          seen = (unsigned)v;
          kind = __ldcg(&s.hc->kind);
          sh.bi[2] = __ldcg(&s.hc->x);
          sh.bi[3] = __ldcg(&s.hc->t);
          sh.bi[4] = __ldcg(&s.hc->b_old);
          sh.bi[5] = __ldcg(&s.hc->ckind);
          sh.bi[6] = __ldcg(&s.hc->cj);
          sh.bi[7] = __ldcg(&s.hc->cmover);
          sh.tmp = __ldcg(&s.hc->ct);
          sh.bd0 = __ldcg(&s.hc->cnewc);
          break;
        }
        if (clock64() - t0 > kSpinLimit) break;
        __nanosleep(64);
      }
      sh.bi[0] = kind;
    }
    __syncthreads();
    const int kind = sh.bi[0];
    if (kind == HJOB_LOG) {
      const unsigned to = (unsigned)sh.bi[1];
      helper_log<NT>(s, applied, to, part, parts);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&s.hc->log_done, to - applied);
      }
      applied = to;
      continue;
    }
    if (kind == HJOB_RELOCATE)
      helper_relocate<NT>(s, sm, pb, sh.bi[2], sh.bi[3], sh.bi[4], part, parts);
    else if (kind == HJOB_CHAIN)
      helper_chain<NT>(s, sh, sh.bi[5], sh.bi[6], sh.bd0, sh.bi[7], sh.tmp, part, parts);
    else
      return;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&s.hc->done, 1u);
    }
  }
}

// Relocation of x from b_old to t through pool slot pos, shared with the
// helper blocks. Block-wide.
template <int NT>
__device__ void relocate_with_helpers(const Scenario& s, Shared& sh, const Smem& sm, int x, int t,
                                      int pos, int b_old) {
  table_sync<NT, true>(s, sh, sm);
  __syncthreads();  // everyone has read the pre-move state
  if (threadIdx.x == 0) {
    s.bveh[b_old] = -1;
    s.bveh[t] = x;
    s.vbase[x] = t;
    sm.gvbase[x] = t;
    s.pkind[pos] = POOL_EMPTY;
    s.pidx[pos] = b_old;
    s.hc->minm = INT_MAX;
    post_job(s, sh, sm, HJOB_RELOCATE, x, t, b_old);
  }
  // meanwhile every other empty row shifts by -D(t, x)
  const long long kt = tix(s, t, x);
  const double At = s.rA[kt], Et = s.rE[kt], Ut = s.rU[kt];
  __syncthreads();  // bveh / vbase updated
  for (int t2 = threadIdx.x; t2 < s.B; t2 += NT) {
    if (s.bveh[t2] >= 0 || t2 == b_old) continue;
    const long long k2 = tix(s, t2, x);
    const int before = table_class(s, sh, t2, x) != CLS_POS;
    const double A = s.rA[k2] - At;
    s.rA[k2] = A;
    s.rE[k2] += Et + 2.0 * kTwoPowM52 * (fabs(At) + fabs(A));
    s.rU[k2] = (s.rU[k2] + Ut) * (1.0 + 2.0 * kTwoPowM52);
    s.rcnt[t2] += (int)(table_class(s, sh, t2, x) != CLS_POS) - before;
  }
  if (threadIdx.x == 0) sh.tmp = 0;
  wait_helpers<NT>(s, sh, sm);
  // the vacated base's fresh row and the imp-row counts
  int cnt = 0;
  for (int v = threadIdx.x; v < s.V; v += NT) {
    const double sum = __ldcg(&s.hsum[v]), abs = __ldcg(&s.habs[v]);
    s.hsum[v] = 0.0;
    s.habs[v] = 0.0;
    const int n = s.vcount[v];
    const long long k = tix(s, b_old, v);
    const double U = abs * (1.0 + (double)(n + 2) * kTwoPowM52);
    s.rA[k] = sum;
    s.rU[k] = U;
    s.rE[k] = (double)(n + 2) * kTwoPowM52 * U;
    cnt += table_class(s, sh, b_old, v) != CLS_POS;
    const int d = __ldcg(&s.hdelta[v]);
    if (d) {
      sm.impc[v] += d;
      s.hdelta[v] = 0;
    }
  }
  if (cnt) atomicAdd(&sh.tmp, cnt);
  __syncthreads();
  if (threadIdx.x == 0) {
    s.rcnt[b_old] = sh.tmp;
    sm.impc[x] = __ldcg(&s.hc->impc_x);
    s.hc->impc_x = 0;
    // the chain's terms changed from the mover's first mission on
    sh.c.hp_valid = min(sh.c.hp_valid, __ldcg(&s.hc->minm) / kChainSub);
  }
  __syncthreads();
}

// ---- moves (proj/src/search.cpp:169-220) ---------------------------------
// Thread 0 only unless noted.

__device__ void set_mission(const Scenario& s, const Smem& sm, int j, int v, double c) {
  s.mv[j] = v;
  s.mc[j] = c;
  const int q = s.invb[j];
  s.mvp[q] = v;
  s.mcp[q] = c;
  if (sm.gmv) {
    sm.gmv[j] = v;
    sm.gmvp[q] = v;
  }
}

// (newc: cost_mb(j, vbase[gain]), already gathered by the caller)
__device__ void apply_takeover(const Scenario& s, Shared& sh, const Smem& sm, int j, int gain,
                               int pos, double newc) {
  const int loser = s.mv[j];
  set_mission(s, sm, j, gain, newc);
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

__device__ void apply_reassign(const Scenario& s, Shared& sh, const Smem& sm, int j, int gain,
                               double newc) {
  const int loser = s.mv[j];
  set_mission(s, sm, j, gain, newc);
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

// Exact accept of a single-substitution candidate (takeover/reassign):
// candidate_total < total, both fixed-order fp64 sums. Block-wide; the new
// exact total is cached when the move is accepted.
template <int NT, bool HELP>
__device__ bool exact_accept_single(const Scenario& s, Shared& sh, const Smem& sm, int j,
                                    double newc) {
  const long long f0 = ph_now();
  const double S = exact_total<NT, HELP>(s, sh, sm);
  const long long c0 = ph_now();
  const double S2 = exact_chain_any<NT, HELP>(s, sh, sm, 1, j, newc, -1, -1, j / kChainSub, 2);
  PH_ADD(sh, 13, c0);
  if (threadIdx.x == 0) {
    sh.c.fallbacks += 1;
    sh.xs = S2;  // the total after the move, if accepted
  }
  PH_ADD(sh, 4, f0);
  __syncthreads();
#ifdef FP_ROW_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0 && sh.c.passes == FP_ROW_TRACE) {
    double q = 0.0, q2 = 0.0;
    for (int k = 0; k < s.M; ++k) {
      q += s.mc[k];
      q2 += k == j ? newc : s.mc[k];
    }
    printf("RT exact j %d S %a S2 %a seqS %a seqS2 %a ver %lld ap %llu\n", j, S, S2, q, q2,
           sh.c.total_ver, (unsigned long long)sh.c.applied);
  }
#endif
  return S2 < S;
}

// Processes the pair (i, j) exactly as try_move x3 (proj/src/search.cpp:277-303,
// 333-341). Block-cooperative; every thread screens each move redundantly
// from the (block-uniform) state, so barriers are only needed around state
// changes and exact sums. Returns with the block synchronised.
template <int NT, bool HELP>
__device__ void process_pair(const Scenario& s, Shared& sh, const Smem& sm, int i, int q,
                             bool tabu, long long tenure, bool debug) {
  // mission j = perm_b[q]; its owner, cost and rotary flag are read from the
  // position-order mirrors (kept in sync on every move), so they do not wait
  // for the perm_b gather
  const int j = sm.pb[q];
  const long long exp = sh.c.tick + tenure;
  // ---- takeover (proj/src/search.cpp:82-101)
  if (i < sh.c.psize && s.pkind[i] == POOL_IDLE) {
    const int g = s.pidx[i];
    const double newc = cost_mb(s, j, s.vbase[g]);
    const double mcj = s.mcp[q];
    if (compat_vm(s.vfixed[g], s.rop[q]) && newc - mcj < 0.0) {
      int acc = mcj - newc > single_bound(s, sh) ? 1 : 0;
      if (!acc) acc = exact_accept_single<NT, HELP>(s, sh, sm, j, newc) ? 3 : 0;
      if (acc) {
        const int loser = s.mvp[q];
        const int nl = s.vcount[loser], ng = s.vcount[g];
        __syncthreads();  // everyone has read the pre-move state
        if (threadIdx.x == 0) {
          apply_takeover(s, sh, sm, j, g, i, newc);
          sh.c.hp_valid = min(sh.c.hp_valid, j / kChainSub);
          sh.c.applied += 1;
          sh.c.pass_applied += 1;
          if (acc == 3) {
            sh.c.total_exact = sh.xs;
            sh.c.total_ver = (long long)sh.c.applied;
          }
          if (tabu) s.exp_take[g] = exp;
          if (debug) debug_check(s, sh);
        }
        // the bit updates read nothing the apply writes (they take the move's
        // new owner and cost as arguments): no barrier in between, except for
        // the debug check and an adopted exact chain
        if (debug || (HELP && acc == 3)) __syncthreads();
        const long long a2 = ph_now();
        bits_after_substitution<NT, HELP>(s, sh, sm, q, j, loser, g, mcj, newc, nl, ng);
        if (HELP && acc == 3) adopt_candidate_sums<NT>(s, sh);
        PH_ADD(sh, 7, a2);
      }
    }
  }
  // ---- relocation (proj/src/search.cpp:103-129), on the state left behind
  if (i < sh.c.psize && s.pkind[i] == POOL_EMPTY) {
    const int t = s.pidx[i];
    const int mover = s.mvp[q];
    if (!(s.vfixed[mover] && s.bheli[t])) {
      relocation_classes<NT, HELP>(s, sh, sm, t);
      const uint8_t cls = sm.cls[mover];
      bool acc = cls == CLS_ACC;
      bool exact_known = false;
      double after = 0.0;
      if (cls == CLS_NEG || cls == CLS_AMB) {
        const long long f0 = ph_now();
        const double* col = s.cost + (long long)t * s.M;
        bool neg = cls == CLS_NEG;
        if (!neg) {
          const long long q0 = ph_now();
          neg = exact_reloc_quick<NT>(s, sh, col, mover, sm.xidx, 2 * NT) < 0.0;
          PH_ADD(sh, 12, q0);
        }
        if (neg) {
          const double S = exact_total<NT, HELP>(s, sh, sm);
          const long long c0 = ph_now();
          after = exact_chain_any<NT, HELP>(s, sh, sm, 2, -1, 0.0, mover, t, 0, 2);
          PH_ADD(sh, 13, c0);
          acc = after < S;
          exact_known = true;
        }
        if (threadIdx.x == 0) sh.c.fallbacks += 1;
        PH_ADD(sh, 4, f0);
      }
      if (acc) {
        const int b_old = s.vbase[mover];
        if (HELP && sm.helpers > 0) {
          const long long a1 = ph_now();
          relocate_with_helpers<NT>(s, sh, sm, mover, t, i, b_old);
          PH_ADD(sh, 6, a1);
        } else {
          const long long a0 = ph_now();
          apply_relocate<NT>(s, sh, mover, t, i);
          if (threadIdx.x == 0) sh.c.hp_valid = 0;
          PH_ADD(sh, 8, a0);
          const long long a1 = ph_now();
          bits_after_relocation<NT>(s, sh, sm, mover, sm.xlist, sm.xlist_cap);
#ifdef FP_RELOC_PROBE
          PH_ADD(sh, 12, a1);
          const long long a2 = ph_now();
#endif
          table_after_relocation<NT>(s, sh, sm, mover, t, b_old);
#ifdef FP_RELOC_PROBE
          PH_ADD(sh, 13, a2);
#endif
          PH_ADD(sh, 6, a1);
        }
        if (threadIdx.x == 0) {
          sh.c.applied += 1;
          sh.c.pass_applied += 1;
          sh.c.pass_relocs += 1;
          if (exact_known) {
            sh.c.total_exact = after;
            sh.c.total_ver = (long long)sh.c.applied;
          }
          if (tabu) {
            // outer {Relocate, target base id} then inner {Relocate, mover id};
            // the second insert wins when the two ids coincide.
            const int ko = s.brk[t], ki = s.vrk[mover];
            s.exp_rel[ko] = exp;
            s.role_rel[ko] = ROLE_OUTER;
            s.exp_rel[ki] = exp;
            s.role_rel[ki] = ROLE_INNER;
            sh.jexp_max = max(sh.jexp_max, exp);
            sh.jkey_ver += 1;
          }
          if (debug) debug_check(s, sh);
        }
        __syncthreads();
        if (HELP && exact_known) adopt_candidate_sums<NT>(s, sh);
      }
    }
  }
  // ---- reassignment (proj/src/search.cpp:131-148)
  {
    const int g = s.mv[i], l = s.mvp[q];
    if (g != l && compat_vm(s.vfixed[g], s.rop[q])) {
      const double newc = cost_mb(s, j, s.vbase[g]);
      const double mcj = s.mcp[q];
      if (newc - mcj < 0.0) {
        int acc = mcj - newc > single_bound(s, sh) ? 1 : 0;
        if (!acc) acc = exact_accept_single<NT, HELP>(s, sh, sm, j, newc) ? 3 : 0;
        if (acc) {
          const int nl = s.vcount[l], ng = s.vcount[g];
          __syncthreads();
          if (threadIdx.x == 0) {
            apply_reassign(s, sh, sm, j, g, newc);
            sh.c.hp_valid = min(sh.c.hp_valid, j / kChainSub);
            sh.c.applied += 1;
            sh.c.pass_applied += 1;
            if (acc == 3) {
              sh.c.total_exact = sh.xs;
              sh.c.total_ver = (long long)sh.c.applied;
            }
            if (tabu) s.exp_reas[g] = exp;
            sh.reassigned = 1;
            if (debug) debug_check(s, sh);
          }
          if (debug || (HELP && acc == 3)) __syncthreads();  // (see the takeover)
          const long long a2 = ph_now();
          bits_after_substitution<NT, HELP>(s, sh, sm, q, j, l, g, mcj, newc, nl, ng);
          if (HELP && acc == 3) adopt_candidate_sums<NT>(s, sh);
          PH_ADD(sh, 7, a2);
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    sh.c.evaluations += 3;
    sh.c.tick += 1;
  }
  __syncthreads();
}

// Row context after any state change, computed by every thread from the
// block-uniform state (no barrier unless a j-key is live or the row
// relocates; those phases publish through shared memory).
struct RowCtx {
  int gain_r, gain_t, rel_t, lim_ro, lim_ra, nj, nrl;
  long long T;  // the tick at the segment start
};

template <int NT, bool HELP>
__device__ RowCtx make_context(const Scenario& s, Shared& sh, const Smem& sm, int i, bool tabu) {
  RowCtx c;
  const long long T = sh.c.tick;
  c.T = T;
  const int g = s.mv[i];
  c.gain_r = g;
  c.gain_t = -1;
  c.rel_t = -1;
  int lim_ro = 0, lim_ra = 0;
  if (i < sh.c.psize) {
    const int k = s.pkind[i], x = s.pidx[i];
    if (k == POOL_IDLE) {
      c.gain_t = x;
      if (tabu) {
        const int lim = clamp_lim(s.exp_take[x] - T, s.M);
        lim_ro = lim;
        lim_ra = lim;
      }
    } else {
      c.rel_t = x;
      if (tabu) {
        const int kk = s.brk[x];
        const int lim = clamp_lim(s.exp_rel[kk] - T, s.M);
        if (s.role_rel[kk] == ROLE_OUTER) lim_ro = lim;
        lim_ra = lim;
      }
    }
  }
  if (tabu) {
    const int lim = clamp_lim(s.exp_reas[g] - T, s.M);
    lim_ro = max(lim_ro, lim);
    lim_ra = max(lim_ra, lim);
  }
  c.lim_ro = lim_ro;
  c.lim_ra = lim_ra;
  c.nj = 0;
  c.nrl = 0;
  __syncwarp();
  if (threadIdx.x == 0) sh.c.counts[2] += 1;
  if (tabu && sh.jexp_max > T) {
    // the vehicles whose {Relocate, id} j-key is live (usually none or a
    // few) with their expiry stamps; rebuilt only after a new insert (a key
    // that has expired since only masks nothing: its window is empty)
    if (sh.jl_ver != sh.jkey_ver) {
      if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        int n = 0;
        for (int v0 = 0; v0 < s.V; v0 += 32) {
          const int v = v0 + l;
          const int k = v < s.V ? s.vrk[v] : 0;
          const long long e = v < s.V ? s.exp_rel[k] : LLONG_MIN;
          const bool live = v < s.V && e > T;
          const unsigned m = __ballot_sync(FULL, live);
          if (live) {
            const int kk = n + __popc(m & ((1u << l) - 1u));
            sm.jl_v[kk] = v;
            sm.jl_exp[kk] = e;
            sm.jl_outer[kk] = s.role_rel[k] == ROLE_OUTER;
          }
          n += __popc(m);
        }
        if (l == 0) {
          sh.nj = n;
          sh.jl_ver = sh.jkey_ver;
        }
      }
      __syncthreads();
    }
    c.nj = sh.nj;
  }
  if (c.rel_t >= 0) {
    relocation_classes<NT, HELP>(s, sh, sm, c.rel_t);
    // the movers that can relocate with gain: the scan's relocation mask is
    // then the OR of their membership words
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      int n = 0;
      for (int v0 = 0; v0 < s.V; v0 += 32) {
        const int v = v0 + l;
        const bool on = v < s.V && sm.cls[v] != CLS_POS;
        const unsigned m = __ballot_sync(FULL, on);
        if (on) sm.rlist[n + __popc(m & ((1u << l) - 1u))] = v;
        n += __popc(m);
      }
      if (l == 0) sh.nrl = n;
    }
    __syncthreads();
    c.nrl = sh.nrl;
  }
  return c;
}

// One outer-index row, proj/src/search.cpp:307-346.
//
// Scan step: the block covers 32*NW words (32 positions each) from the
// current position. Per word (one lane): candidates = imp[gain of the row]
// | imp[idle pool vehicle] | relocation mask; blocked = row-key prefix |
// the positions of vehicles whose j-key is live (mem rows, within their live
// windows); outer = row outer prefix | outer j-key positions. The first event
// is the first set bit of outer | (candidates & ~blocked); the positions
// before it are either inner-blocked (tick + skip) or evaluated (3
// evaluations each), counted with popc.
template <int NT, bool HELP>
__device__ void run_row(const Scenario& s, Shared& sh, const Smem& sm, int i, bool tabu,
                        long long tenure, bool debug) {
  constexpr int NW = NT / 32;
  const int M = s.M, nwd = s.nwd;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int p = 0;
  int parity = 0;
  if (threadIdx.x == 0) sh.c.counts[0] += 1;
  while (p < M) {
    const long long c0 = ph_now();
    const RowCtx cx = make_context<NT, HELP>(s, sh, sm, i, tabu);
    PH_ADD(sh, 1, c0);
    const long long c1 = ph_now();
    const int p_seg = p;
    const int gain_r = cx.gain_r, gain_t = cx.gain_t, rel_t = cx.rel_t;
    const int lim_ro = cx.lim_ro, lim_ra = cx.lim_ra, nj = cx.nj;
    const int nrl = cx.nrl;
    const uint32_t* imp_r = s.imp + (long long)gain_r * nwd;
    const uint32_t* imp_t = s.imp + (long long)(gain_t >= 0 ? gain_t : 0) * nwd;
    int ev = INT_MAX;
    while (p < M) {
      const int w0 = p >> 5;
      const int wd = w0 + w * 32 + l;
      const long long base = (long long)wd * 32;
      uint32_t relw = 0;
      if (rel_t >= 0 && nrl <= 8) {
        // relocation candidates: the positions of the few movers that can gain
        // (unrolled: the membership words' gathers are in flight together)
        if (wd < nwd)
#pragma unroll 4
          for (int k = 0; k < nrl; ++k) relw |= s.mem[(long long)sm.rlist[k] * nwd + wd];
      } else if (rel_t >= 0) {
        // many movers: the vehicle of every position, one coalesced pass over
        // the warp's 32 words, lane = position
        for (int k = 0; k < 32; ++k) {
          const long long q = (long long)(w0 + w * 32 + k) * 32 + l;
          bool b = false;
          if (q < M && q >= p) b = sm.cls[s.mvp[q]] != CLS_POS;
          const unsigned m = __ballot_sync(FULL, b);
          if (l == k) relw = m;
        }
      }
      uint32_t valid = 0, evw = 0, blk = 0;
      if (wd < nwd) {
        valid = prefix_bits(M - base) & ~prefix_bits(p - base);
        uint32_t cand = imp_r[wd] | relw;
        if (gain_t >= 0) cand |= imp_t[wd];
        uint32_t outer = 0;
        if (tabu) {
          outer = prefix_bits(p_seg + lim_ro - base);
          blk = prefix_bits(p_seg + lim_ra - base);
#pragma unroll 4
          for (int k = 0; k < nj; ++k) {
            const uint32_t m =
                s.mem[(long long)sm.jl_v[k] * nwd + wd] &
                prefix_bits(p_seg + clamp_lim(sm.jl_exp[k] - cx.T, M) - base);
            blk |= m;
            if (sm.jl_outer[k]) outer |= m;
          }
          outer &= valid;
          blk = (blk | outer) & valid;
        }
        evw = outer | (cand & ~blk & valid);
      }
      // warp: first event and the counts before it
      const unsigned evl = __ballot_sync(FULL, evw != 0u);
      int n_valid, n_blk, evpos = INT_MAX;
      if (evl) {
        const int f = __ffs(evl) - 1;
        if (l < f) {
          n_valid = __popc(valid);
          n_blk = __popc(blk);
        } else if (l == f) {
          const int bn = __ffs(evw) - 1;
          const uint32_t below = (1u << bn) - 1u;
          n_valid = __popc(valid & below);
          n_blk = __popc(blk & below);
          evpos = (int)(base + bn);
        } else {
          n_valid = 0;
          n_blk = 0;
        }
      } else {
        n_valid = __popc(valid);
        n_blk = __popc(blk);
      }
      n_valid = (int)__reduce_add_sync(FULL, (unsigned)n_valid);
      n_blk = (int)__reduce_add_sync(FULL, (unsigned)n_blk);
      evpos = __reduce_min_sync(FULL, evpos);
      // one barrier per step: summaries are double-buffered by step parity and
      // every warp combines them itself (no broadcast round)
      int* ws = sm.wsum + (parity & 1) * NW * 3;
      parity ^= 1;
      if (l == 0) {
        ws[w * 3 + 0] = evpos;
        ws[w * 3 + 1] = n_valid;
        ws[w * 3 + 2] = n_blk;
      }
      __syncthreads();
      const int e = l < NW ? ws[l * 3 + 0] : INT_MAX;
      int nv = l < NW ? ws[l * 3 + 1] : 0;
      int nb = l < NW ? ws[l * 3 + 2] : 0;
      const unsigned any = __ballot_sync(FULL, e != INT_MAX);
      const int wstar = any ? __ffs(any) - 1 : 32;
      if (l > wstar) {
        nv = 0;
        nb = 0;
      }
      nv = (int)__reduce_add_sync(FULL, (unsigned)nv);
      nb = (int)__reduce_add_sync(FULL, (unsigned)nb);
      ev = any ? __shfl_sync(FULL, e, wstar) : INT_MAX;
      if (threadIdx.x == 0) {
        sh.c.counts[1] += 1;
        sh.c.skips_inner += (unsigned long long)nb;
        sh.c.evaluations += 3ull * (unsigned long long)(nv - nb);
        if (tabu) sh.c.tick += nv;  // every position before the event is one pair
        if (nb > 0) sh.c.pass_skipped = 1;
      }
      p = ev != INT_MAX ? ev : (int)min((long long)M, (long long)(w0 + 32 * NW) * 32);
      if (ev != INT_MAX) break;
    }
    PH_ADD(sh, 2, c1);
    if (ev == INT_MAX) return;  // row exhausted perm_b
    // event at position p
    bool outer_ev = false;
    if (tabu) {
      const int off = p - p_seg;
      outer_ev = off < lim_ro;
      if (!outer_ev && nj > 0) {
        const int v = s.mvp[p];
        const int kk = s.vrk[v];
        outer_ev = off < clamp_lim(s.exp_rel[kk] - cx.T, s.M) && s.role_rel[kk] == ROLE_OUTER;
      }
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
    if (threadIdx.x == 0) sh.reassigned = 0;
#ifdef FP_ROW_TRACE
    const unsigned long long tr_ap = sh.c.applied;
    if (threadIdx.x == 0 && blockIdx.x == 0 && sh.c.passes == FP_ROW_TRACE) {
      const int j = sm.pb[p], g = s.mv[i], l = s.mv[j];
      printf("RT pre i %d p %d j %d g %d l %d vb %d newc %a mcj %a mcp %a mvp %d tu %a ps %d vf %d ro %d sb %a fe %d\n", i, p, j, g, l,
             s.vbase[g], cost_mb(s, j, s.vbase[g]), s.mc[j], s.mcp[p], s.mvp[p], sh.c.total_up, sh.c.psize,
             (int)s.vfixed[g], (int)s.ro[j], single_bound(s, sh), sh.c.force_exact);
    }
#endif
    process_pair<NT, HELP>(s, sh, sm, i, p, tabu, tenure, debug);
#ifdef FP_ROW_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0 && sh.c.passes == FP_ROW_TRACE)
      printf("RT pair i %d p %d j %d applied %d fb %llu ev %llu\n", i, p, s.mvp[p] , (int)(sh.c.applied - tr_ap),
             (unsigned long long)sh.c.fallbacks, (unsigned long long)sh.c.evaluations);
#endif
    PH_ADD(sh, 3, c2);
    if (sh.c.error) return;
    p += 1;
    if (tabu && tenure > 1 && sh.reassigned && p < M) {
      // the reassignment just inserted {Reassign, id(vehicle(i))} with the
      // Outer role and expiry tick + tenure: the row's next pair checks that
      // key, finds it live (tenure > 1) and ends the row there -- one tick,
      // one outer skip (proj/src/search.cpp:312-330), no context or scan
      if (threadIdx.x == 0) {
        sh.c.skips_outer += 1;
        sh.c.tick += 1;
        sh.c.pass_skipped = 1;
      }
      __syncthreads();
      return;
    }
  }
}

__host__ __device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

// 32 x 32 bit-matrix transpose across a warp: lane r holds row r (bit c =
// column c); afterwards lane c holds column c (bit r = row r). Five
// shuffle-exchange stages swapping the off-diagonal j x j blocks.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  uint32_t m = 0x0000FFFFu;
#pragma unroll
  for (int j = 16; j != 0; j >>= 1, m ^= (m << j)) {
    const uint32_t y = __shfl_xor_sync(FULL, x, j);
    if ((lane & j) == 0) {
      x ^= (((x >> j) ^ y) & m) << j;
    } else {
      x ^= ((y >> j) ^ x) & m;
    }
  }
  return x;
}

// Per pass: the perm_b-ordered mirrors and the imp/mem bitsets, warp per
// word, lane per position: each lane gathers its mission's natural-order
// improvement row (NVW words) and the warp transposes it into the V
// position-order words with ballots; mem from the mirrored vehicles.
__device__ void prep_words(const Scenario& s, const int32_t* __restrict__ pb, int wd0, int wstride) {
#ifndef FP_PREP_UW
#define FP_PREP_UW 4
#endif
  constexpr int UW = FP_PREP_UW;  // words per warp iteration: their loads in flight together
  const int l = threadIdx.x & 31;
  const int nvw = s.nvw, V = s.V;
  for (int wb = wd0; wb < s.nwd; wb += wstride * UW) {
    int j[UW], v[UW];
    bool valid[UW];
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int wd = wb + u * wstride;
      const int q = wd * 32 + l;
      valid[u] = wd < s.nwd && q < s.M;
      j[u] = valid[u] ? pb[q] : 0;
    }
    double mcv[UW];
    uint8_t rov[UW];
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      v[u] = valid[u] ? s.mv[j[u]] : -1;
      mcv[u] = valid[u] ? s.mc[j[u]] : 0.0;
      rov[u] = valid[u] ? s.ro[j[u]] : 0;
    }
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      if (valid[u]) {
        const int q = (wb + u * wstride) * 32 + l;
        s.mvp[q] = v[u];
        s.mcp[q] = mcv[u];
        s.rop[q] = rov[u];
        s.invb[j[u]] = q;
      }
    }
    // per vehicle word: the 32 lanes' rows form a 32 x 32 bit matrix; its
    // transpose gives lane b the position word of vehicle 32*vw + b
    for (int vw = 0; vw < nvw; ++vw) {
      const int g = vw * 32 + l;
      uint32_t rows[UW];
#pragma unroll
      for (int u = 0; u < UW; ++u) rows[u] = valid[u] ? s.impT[(long long)j[u] * nvw + vw] : 0u;
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int wd = wb + u * wstride;
        if (wd >= s.nwd) break;
        const uint32_t row = rows[u];
        const int dv = v[u] - vw * 32;
        const uint32_t one = (dv >= 0 && dv < 32) ? 1u << dv : 0u;
        const uint32_t it = transpose32(row, l), mt = transpose32(one, l);
        if (g < V) {
          s.imp[(long long)g * s.nwd + wd] = it;
          s.mem[(long long)g * s.nwd + wd] = mt;
        }
      }
    }
  }
}

// Test hook (Counters::check_impt): every natural-order improvement row
// against the table. Block-wide; sets error 6 on a mismatch.
template <int NT>
__device__ void verify_impt(const Scenario& s, Shared& sh) {
  if (threadIdx.x == 0) sh.tmp = 0;
  __syncthreads();
  int bad = 0;
  for (int j = threadIdx.x; j < s.M; j += NT) {
    for (int vw = 0; vw < s.nvw; ++vw) {
      uint32_t row = 0;
      for (int b = 0; b < 32 && vw * 32 + b < s.V; ++b) {
        const int g = vw * 32 + b;
        const bool on = s.mv[j] != g && compat_vm(s.vfixed[g], s.ro[j]) &&
                        cost_at(s, s.vbase[g], j) < s.mc[j];
        row |= (uint32_t)on << b;
      }
      bad |= row != s.impT[(long long)j * s.nvw + vw];
    }
  }
  if (bad) atomicOr(&sh.tmp, 1);
  __syncthreads();
  if (threadIdx.x == 0 && sh.tmp) sh.c.error = 6;
  __syncthreads();
}

// grid = (words, scenarios): the sweep for large scenarios, one launch per pass.
__global__ void __launch_bounds__(256) prep_kernel(Scenario* scs, const int32_t* __restrict__ active,
                                                   const int32_t* __restrict__ pb) {
  if (!active[blockIdx.y]) return;
  const Scenario s = scs[blockIdx.y];
  if (s.ctr->done) return;  // finished earlier in this chunk of launches
  const int warps = blockDim.x >> 5;
  prep_words(s, pb, blockIdx.x * warps + (threadIdx.x >> 5), gridDim.x * warps);
}

// Block-wide copy of n words from global memory into shared memory (both
// 16-byte aligned): four 16-byte loads in flight per thread.
template <int NT>
__device__ void copy_words(uint32_t* dst, const uint32_t* __restrict__ src, long long n) {
  const long long n4 = n >> 2;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (long long k0 = 0; k0 < n4; k0 += 4ll * NT) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long k = k0 + u * NT + threadIdx.x;
      if (k < n4) r[u] = __ldg(s4 + k);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long k = k0 + u * NT + threadIdx.x;
      if (k < n4) d4[k] = r[u];
    }
  }
  for (long long k = (n4 << 2) + threadIdx.x; k < n; k += NT) dst[k] = src[k];
}

// Shared-memory bytes of the always-resident part and of the optional copy
// of the small per-vehicle / per-key state.
size_t pass_smem_core(int V, int NT) {
  const int NW = NT / 32;
  return align16(4ull * V) + align16(V) + align16(V) + 2 * align16(8ull * NW * V) +
         align16(8ull * NW * 32) + align16(8ull * NW * 3) + 3 * align16(4ull * V) + align16(V) +
         align16(8ull * NT) + align16(8ull * NT) + 2 * align16(4ull * V) + 64;
}
size_t pass_smem_state(int V, int B, int K) {
  return align16(8ull * V) * 2 + align16(8ull * K) + align16(K) + align16(4ull * V) * 3 +
         align16(V) + 2 * align16(4ull * B) + align16(B) + 64;
}

// One pass over perm_a for every active scenario (blockIdx.x = scenario).
// INK: the block rebuilds its own mirrors / bitsets between passes (a
// separate instantiation, so the grid-wide-sweep variant carries none of
// that code's registers).
template <int NT, bool INK, bool HELP>
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : (NT == 256 ? 2 : 4))
    pass_kernel(Scenario* scs, const int32_t* __restrict__ active, const int32_t* __restrict__ perms,
                int kpasses, int inkernel_prep, int max_passes, int tabu_i, long long tenure,
                int debug_i, int state_in_smem, int bits_in_smem, int mirrors_in_smem,
                int helpers, unsigned epoch, const int* __restrict__ perm_bad) {
  // a rejected draw in the device permutation stream: the host redoes the chunk
  if (perm_bad && *perm_bad) return;
  // with helpers the grid is one scenario: block 0 runs it, the others help
  const int scn = helpers > 0 ? 0 : blockIdx.x;
  if (!active[scn]) return;
  const Scenario g = scs[scn];
  if (g.ctr->done) return;  // finished earlier in this chunk of launches
  const long long t_entry = clock64();  // phase 15: the whole launch (block 0's SM clock)
  Scenario s = g;
  // the scenario's own SearchConfig and permutation stream (a chunk holds
  // 2 * kpasses permutations per stream, stream after stream)
  (void)tabu_i;
  (void)debug_i;
  const bool tabu = g.tabu != 0, debug = g.debug != 0;
  tenure = g.tenure;
  max_passes = g.max_passes;
  perms += (long long)g.pstream * 2ll * kpasses * g.M;
  __shared__ Shared sh;
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr int NW = NT / 32;
  const int V = s.V, B = s.B, K = s.K;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = dyn + off;
    off = align16(off + bytes);
    return p;
  };
  Smem sm;
  sm.lim_j = reinterpret_cast<int*>(take(4ull * V));
  sm.outer_j = take(V);
  sm.cls = take(V);
  sm.acc_sum = reinterpret_cast<double*>(take(8ull * NW * V));
  sm.acc_abs = reinterpret_cast<double*>(take(8ull * NW * V));
  sm.stage = reinterpret_cast<double*>(take(8ull * NW * 32));
  sm.wsum = reinterpret_cast<int*>(take(8ull * NW * 3));
  sm.xidx = reinterpret_cast<int*>(take(8ull * NT));
  sm.xlist = s.scratch;
  sm.xlist_cap = s.M;
  sm.jl_v = reinterpret_cast<int*>(take(4ull * V));
  sm.jl_exp = reinterpret_cast<long long*>(take(8ull * V));
  sm.jl_outer = take(V);
  sm.impc = reinterpret_cast<int*>(take(4ull * V));
  sm.rlist = reinterpret_cast<int*>(take(4ull * V));
  sm.paw = reinterpret_cast<int*>(take(8ull * NT));
  sm.pb = perms + s.M;
  sm.helpers = helpers;
  sm.epoch = epoch;
  sm.gvbase = g.vbase;
  sm.gmv = nullptr;
  sm.gmvp = nullptr;
  if (HELP && helpers > 0 && blockIdx.x > 0) {
    helper_loop<NT>(g, sh, sm, perms + s.M, blockIdx.x - 1, helpers);
    return;
  }
  if (state_in_smem) {
    // the small mutable state lives in shared memory for the whole pass
    s.exp_take = reinterpret_cast<long long*>(take(8ull * V));
    s.exp_reas = reinterpret_cast<long long*>(take(8ull * V));
    s.exp_rel = reinterpret_cast<long long*>(take(8ull * K));
    s.role_rel = take(K);
    s.vbase = reinterpret_cast<int32_t*>(take(4ull * V));
    s.vcount = reinterpret_cast<int32_t*>(take(4ull * V));
    int32_t* vrk = reinterpret_cast<int32_t*>(take(4ull * V));
    uint8_t* vfixed = take(V);
    int32_t* brk = reinterpret_cast<int32_t*>(take(4ull * B));
    uint8_t* bheli = take(B);
    s.bveh = reinterpret_cast<int32_t*>(take(4ull * B));
    for (int v = threadIdx.x; v < V; v += NT) {
      s.exp_take[v] = g.exp_take[v];
      s.exp_reas[v] = g.exp_reas[v];
      s.vbase[v] = g.vbase[v];
      s.vcount[v] = g.vcount[v];
      vrk[v] = g.vrk[v];
      vfixed[v] = g.vfixed[v];
    }
    for (int k = threadIdx.x; k < K; k += NT) {
      s.exp_rel[k] = g.exp_rel[k];
      s.role_rel[k] = g.role_rel[k];
    }
    for (int b = threadIdx.x; b < B; b += NT) {
      brk[b] = g.brk[b];
      bheli[b] = g.bheli[b];
      s.bveh[b] = g.bveh[b];
    }
    s.vrk = vrk;
    s.vfixed = vfixed;
    s.brk = brk;
    s.bheli = bheli;
  }
  if (bits_in_smem) {
    // the imp / mem bitsets live in shared memory: every scan step, event
    // and bit update of the pass then stays on the SM
    s.imp = reinterpret_cast<uint32_t*>(take(4ull * V * s.nwd));
    s.mem = reinterpret_cast<uint32_t*>(take(4ull * V * s.nwd));
  }
  if (mirrors_in_smem) {
    // mission -> vehicle (both orders), the pool and the unsettled-row counts
    // in shared memory too; mv / mvp are written through (the sweep and the
    // helpers read them), the rest is written back at the end. With helper
    // blocks patching a large table (B > NT, the patch log) the unsettled-row
    // counts stay in global memory: the helpers update them.
    s.mv = reinterpret_cast<int32_t*>(take(4ull * s.M));
    s.mvp = reinterpret_cast<int32_t*>(take(4ull * s.M));
    s.pkind = reinterpret_cast<int32_t*>(take(4ull * s.pool_cap));
    s.pidx = reinterpret_cast<int32_t*>(take(4ull * s.pool_cap));
    int32_t* rc = reinterpret_cast<int32_t*>(take(4ull * B));
    if (helpers == 0 || B <= NT) s.rcnt = rc;
    sm.gmv = g.mv;
    sm.gmvp = g.mvp;
    copy_words<NT>(reinterpret_cast<uint32_t*>(s.mv), reinterpret_cast<const uint32_t*>(g.mv), s.M);
    for (int k = threadIdx.x; k < s.pool_cap; k += NT) {
      s.pkind[k] = g.pkind[k];
      s.pidx[k] = g.pidx[k];
    }
    if (helpers == 0 || B <= NT)
      for (int b = threadIdx.x; b < B; b += NT) s.rcnt[b] = g.rcnt[b];
  }
  if (threadIdx.x == 0) {
    sh.c = *s.ctr;
    sh.jexp_max = LLONG_MIN;
    sh.jkey_ver = 0;
    sh.jl_ver = -1;
    sh.hk = 0;
    sh.hdone = helpers > 0 ? s.hc->done : 0u;
    sh.lt = 0;
    sh.lsync = 0;
    sh.hp2_from = -1;
    sh.ldone0 = helpers > 0 ? s.hc->log_done : 0u;
  }
  __syncthreads();
  {
    // latest vehicle j-key expiry (maintained on inserts afterwards)
    const int l = threadIdx.x & 31;
    long long e = LLONG_MIN;
    for (int v = threadIdx.x; v < V; v += NT) e = max(e, s.exp_rel[s.vrk[v]]);
    for (int o = 16; o > 0; o >>= 1) e = max(e, __shfl_xor_sync(FULL, e, o));
    if (l == 0) atomicMax(&sh.jexp_max, e);
  }
  __syncthreads();
  const int M = s.M;
  for (int kp = 0; kp < kpasses && !sh.c.done; ++kp) {
    const int32_t* pa = perms + 2ll * kp * M;
    sm.pb = pa + M;
    const long long ps0 = ph_now();
    if (sh.c.check_impt) verify_impt<NT>(s, sh);
    if (INK) {
      prep_words(s, sm.pb, threadIdx.x >> 5, NW);
      __syncthreads();
    } else if (bits_in_smem || mirrors_in_smem) {
      // the grid-wide sweep built them in global memory: 16-byte loads, a
      // batch of them in flight per thread before any store
      if (bits_in_smem) {
        copy_words<NT>(s.imp, g.imp, (long long)V * s.nwd);
        copy_words<NT>(s.mem, g.mem, (long long)V * s.nwd);
      }
      if (mirrors_in_smem)
        copy_words<NT>(reinterpret_cast<uint32_t*>(s.mvp), reinterpret_cast<const uint32_t*>(g.mvp),
                       s.M);
      __syncthreads();
    }
    {
      // imp row popcounts (warp per vehicle)
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      for (int v = w; v < V; v += NW) {
        int c = 0;
        for (int wd = l; wd < s.nwd; wd += 32) c += __popc(s.imp[(long long)v * s.nwd + wd]);
        c = (int)__reduce_add_sync(FULL, (unsigned)c);
        if (l == 0) sm.impc[v] = c;
      }
    }
    if (threadIdx.x == 0) {
      sh.c.pass_applied = 0;
      sh.c.pass_relocs = 0;
      sh.c.pass_skipped = 0;
    }
    __syncthreads();
    PH_ADD(sh, 11, ps0);
    int r = 0;
    int pw = INT_MIN;  // perm_a window in shared memory: sm.paw[k] = pa[pw + k], k < 2*NT
    int par = 0;       // parity of the double-buffered row-run reduction
    long long T = sh.c.tick;  // every thread tracks the tick through row runs
    while (r < M && !sh.c.error) {
      const long long b0 = ph_now();
      // relocation-table patches published to the helper blocks and not yet
      // confirmed: instead of waiting for them here, a row whose eventless
      // test needs rcnt (its pool entry is an empty base) counts as
      // nontrivial -- run_row settles it exactly after its own table_sync --
      // so the patches overlap the classification of the rows that follow
      const bool patches_pending = HELP && sm.helpers > 0 && sh.lt != sh.lsync;
      if (r < pw || r + NT > pw + 2 * NT) {
        pw = r;
        for (int k = threadIdx.x; k < 2 * NT; k += NT) sm.paw[k] = pw + k < M ? pa[pw + k] : 0;
        __syncthreads();
      }
      // Classify the next NT rows at the current tick T (thread d: row r+d):
      //  S: no move from its outer index can improve any mission (imp rows
      //     empty, relocation classes all POS) -- tick independent;
      //  F: latest expiry of any key that could touch the row (row keys and
      //     every vehicle's {Relocate, id} j-key); F <= T: none ever live again;
      //  E: expiry of its keys that block pair 0 with the Outer role.
      // A row with S and F <= T is eventless at any later tick: all M pairs
      // are evaluated (M ticks, 3M evaluations). A row with T_d < E is
      // outer-blocked at its first pair (1 tick).
      const int d = threadIdx.x, row = r + d;
      int first_nontrivial = INT_MAX, first_nonouter = INT_MAX;
      if (row < M) {
        const int i = sm.paw[row - pw];
        const int g0 = s.mv[i];
        bool st = sm.impc[g0] == 0;
        long long F = tabu ? max(s.exp_reas[g0], sh.jexp_max) : LLONG_MIN;
        long long E = tabu ? s.exp_reas[g0] : LLONG_MIN;
        if (i < sh.c.psize) {
          const int x = s.pidx[i];
          if (s.pkind[i] == POOL_IDLE) {
            st = st && sm.impc[x] == 0;
            if (tabu) {
              F = max(F, s.exp_take[x]);
              E = max(E, s.exp_take[x]);
            }
          } else {
            st = st && !patches_pending && s.rcnt[x] == 0;
            if (tabu) {
              const int k = s.brk[x];
              F = max(F, s.exp_rel[k]);
              if (s.role_rel[k] == ROLE_OUTER) E = max(E, s.exp_rel[k]);
            }
          }
        }
        if (tabu) {
          const int k = s.vrk[s.mvp[0]];
          if (s.role_rel[k] == ROLE_OUTER) E = max(E, s.exp_rel[k]);
        }
        if (!(st && F <= T)) first_nontrivial = d;
        if (!(T + d < E)) first_nonouter = d;
      }
      // both block minima with one barrier (double-buffered by parity; every
      // warp combines the per-warp values itself)
      {
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        const int a = __reduce_min_sync(FULL, first_nontrivial);
        const int o = __reduce_min_sync(FULL, first_nonouter);
        if (l == 0) {
          sh.red2[par][w][0] = a;
          sh.red2[par][w][1] = o;
        }
        __syncthreads();
        first_nontrivial = l < NT / 32 ? sh.red2[par][l][0] : INT_MAX;
        first_nonouter = l < NT / 32 ? sh.red2[par][l][1] : INT_MAX;
        first_nontrivial = __reduce_min_sync(FULL, first_nontrivial);
        first_nonouter = __reduce_min_sync(FULL, first_nonouter);
        par ^= 1;
      }
      const int A = first_nontrivial;
      if (A > 0) {
        // a run of eventless rows
        const int n = A == INT_MAX ? min(NT, M - r) : A;
        if (threadIdx.x == 0) {
          sh.c.evaluations += 3ull * (unsigned long long)M * (unsigned long long)n;
          if (tabu) sh.c.tick += (long long)M * n;
          sh.c.counts[4] += (unsigned long long)n;
        }
        if (tabu) T += (long long)M * n;
#ifdef FP_ROW_TRACE
        if (threadIdx.x == 0 && blockIdx.x == 0 && sh.c.passes == FP_ROW_TRACE)
          printf("RT run %d %d E\n", r, n);
#endif
        r += n;
        PH_ADD(sh, 0, b0);
        continue;
      }
      if (tabu) {
        // a run of rows outer-blocked at their first pair (one tick each)
        const int nskip = first_nonouter == INT_MAX ? min(NT, M - r) : first_nonouter;
        if (threadIdx.x == 0 && nskip > 0) {
          sh.c.tick += nskip;
          sh.c.skips_outer += (unsigned long long)nskip;
          sh.c.pass_skipped = 1;
        }
        T += nskip;
#ifdef FP_ROW_TRACE
        if (threadIdx.x == 0 && blockIdx.x == 0 && sh.c.passes == FP_ROW_TRACE && nskip > 0)
          printf("RT run %d %d O\n", r, nskip);
#endif
        r += nskip;
        PH_ADD(sh, 0, b0);
        if (nskip > 0) continue;
      }
      // (the reduction barrier above published thread 0's counter updates)
      run_row<NT, HELP>(s, sh, sm, sm.paw[r - pw], tabu, tenure, debug);
      __syncthreads();
#ifdef FP_ROW_TRACE
      if (threadIdx.x == 0 && blockIdx.x == 0 && sh.c.passes == FP_ROW_TRACE)
        printf("RT row %d i %d ev %llu tick %lld so %llu si %llu ap %d\n", r, sm.paw[r - pw],
               (unsigned long long)sh.c.evaluations, (long long)sh.c.tick,
               (unsigned long long)sh.c.skips_outer, (unsigned long long)sh.c.skips_inner,
               (int)sh.c.pass_applied);
#endif
      T = sh.c.tick;
      r += 1;
    }
    table_sync<NT, HELP>(s, sh, sm);  // the next launch starts from a complete table
    // end of pass: run_search's keep_going / max_passes (search.cpp:420-428)
    if (threadIdx.x == 0) {
      sh.c.passes += 1;
      const bool keep = sh.c.error == 0 &&
                        (sh.c.pass_applied > 0 || (tabu && sh.c.pass_skipped));
      if (!keep || (max_passes >= 0 && sh.c.passes >= max_passes)) sh.c.done = 1;
    }
    __syncthreads();
  }
  if (state_in_smem) {
    for (int v = threadIdx.x; v < V; v += NT) {
      g.exp_take[v] = s.exp_take[v];
      g.exp_reas[v] = s.exp_reas[v];
      g.vbase[v] = s.vbase[v];
      g.vcount[v] = s.vcount[v];
    }
    for (int k = threadIdx.x; k < K; k += NT) {
      g.exp_rel[k] = s.exp_rel[k];
      g.role_rel[k] = s.role_rel[k];
    }
    for (int b = threadIdx.x; b < B; b += NT) g.bveh[b] = s.bveh[b];
  }
  if (mirrors_in_smem) {
    for (int k = threadIdx.x; k < s.pool_cap; k += NT) {
      g.pkind[k] = s.pkind[k];
      g.pidx[k] = s.pidx[k];
    }
    if (helpers == 0 || B <= NT)
      for (int b = threadIdx.x; b < B; b += NT) g.rcnt[b] = s.rcnt[b];
  }
  if (threadIdx.x == 0) {
    sh.c.cycles[15] += (unsigned long long)(clock64() - t_entry);
    *g.ctr = sh.c;
  }
  if (helpers > 0) {
    __syncthreads();
    if (threadIdx.x == 0) post_job(s, sh, sm, HJOB_QUIT, -1, -1, -1);
  }
}

// The row-major copy of a column-major table: 32-base x 64-mission tiles
// through shared memory, eight 8-byte loads in flight per thread, 256-byte
// coalesced rows on both sides.
__device__ __forceinline__ void transpose_tile(const double* __restrict__ src, int M, int B,
                                               double* __restrict__ dst, int m0, int b0) {
  __shared__ double tile[32][65];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int b = b0 + ty + 8 * (r >> 1), m = m0 + tx + 32 * (r & 1);
    v[r] = (b < B && m < M) ? src[(long long)b * M + m] : 0.0;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) tile[ty + 8 * (r >> 1)][tx + 32 * (r & 1)] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int m = m0 + ty + 8 * r, b = b0 + tx;
    if (m < M && b < B) dst[(long long)m * B + b] = tile[tx][ty + 8 * r];
  }
}

__global__ void __launch_bounds__(256) transpose_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.z];
  const int m0 = blockIdx.x * 64, b0 = blockIdx.y * 32;
  if (!s.costT || m0 >= s.M || b0 >= s.B) return;
  transpose_tile(s.cost, s.M, s.B, const_cast<double*>(s.costT), m0, b0);
}

__global__ void __launch_bounds__(256) transpose_table_kernel(const double* __restrict__ src, int M,
                                                              int B, double* __restrict__ dst) {
  transpose_tile(src, M, B, dst, blockIdx.x * 64, blockIdx.y * 32);
}

cudaError_t launch_transpose(const double* src, int M, int B, double* dst, cudaStream_t stream) {
  if (M > 0 && B > 0)
    transpose_table_kernel<<<dim3((M + 63) / 64, (B + 31) / 32), 256, 0, stream>>>(src, M, B, dst);
  return cudaGetLastError();
}

// Search start, part 1: per-mission costs (SearchState::from,
// proj/src/search.cpp:41-48), grid-wide (blockIdx.y = scenario).
__global__ void __launch_bounds__(256) mission_cost_kernel(Scenario* scs) {
  const Scenario& s = scs[blockIdx.y];
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < s.M; m += gridDim.x * blockDim.x)
    s.mc[m] = cost_at(s, s.vbase[s.mv[m]], m);
}

// Search start, part 2: the exact initial fixed-order total, one block per
// scenario (the block-parallel integer-binade chain).
__global__ void __launch_bounds__(512) init_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.x];
  __shared__ Shared sh;
  const double t = exact_chain<512>(s, sh, 0, -1, 0.0, -1, nullptr);
  if (threadIdx.x == 0) {
    s.ctr->total_up = t;
    s.ctr->final_total = t;
    s.ctr->total_exact = t;
    s.ctr->total_ver = 0;
  }
}

// The natural-order improvement rows at the search start, thread per
// mission: every occupied vehicle's base column streamed once, coalesced
// (V*M table reads; the neighbourhood evaluation of every reassignment).
__global__ void __launch_bounds__(256) impt_init_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.y];
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= s.M) return;
  const int v = s.mv[j];
  const double mcj = s.mc[j];
  const bool ro = s.ro[j];
  for (int vw = 0; vw < s.nvw; ++vw) {
    uint32_t row = 0;
    const int gend = min(32, s.V - vw * 32);
#pragma unroll 8
    for (int b = 0; b < gend; ++b) {
      const int g = vw * 32 + b;
      const bool on = v != g && compat_vm(s.vfixed[g], ro) && cost_at(s, s.vbase[g], j) < mcj;
      row |= (uint32_t)on << b;
    }
    s.impT[(long long)j * s.nvw + vw] = row;
  }
}

// The relocation-delta table's initial rows, one block per empty base (the
// sweep over every empty base's column: 8*M bytes each, streamed coalesced).
__global__ void __launch_bounds__(256) table_rows_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.y];
  const int t = blockIdx.x;
  if (t >= s.B || s.bveh[t] >= 0) return;
  __shared__ Shared sh;
  extern __shared__ __align__(16) unsigned char dyn[];
  double* acc_sum = reinterpret_cast<double*>(dyn);
  double* acc_abs = acc_sum + 8 * s.V;
  double* stage = acc_abs + 8 * s.V;
  if (threadIdx.x == 0) sh.c = *s.ctr;
  __syncthreads();
  table_row_fresh<256>(s, sh, acc_sum, acc_abs, stage, t);
}

// ---- relocation-table build from the row-major copy (single scenario) ----
// D(t, v) for every base t at once: a block takes a chunk of vehicle v's
// missions and streams their rows of the row-major table (B contiguous
// costs each), thread per base with register accumulators; chunks combine
// with fp64 atomics (any order: the table's bounds hold for any summation
// order). HBM-bound: every table entry is read once, coalesced.

// Plan: per-vehicle segment starts and the chunk list. One thread.
__global__ void rows_plan_kernel(Scenario* scs) {
  const Scenario s = scs[0];
  if (threadIdx.x != 0) return;
  int off = 0, nc = 0;
  for (int v = 0; v < s.V; ++v) {
    s.vseg[v] = off;
    s.vcur[v] = off;
    const int c = s.vcount[v];
    for (int k = 0; k < c; k += kRowsChunk) {
      s.vch[3 * nc] = v;
      s.vch[3 * nc + 1] = off + k;
      s.vch[3 * nc + 2] = off + min(c, k + kRowsChunk);
      ++nc;
    }
    off += c;
  }
  s.vseg[s.V] = off;
  s.vseg[s.V + 1] = nc;
}

// Missions grouped by vehicle into scratch (order inside a group is free).
__global__ void __launch_bounds__(256) rows_group_kernel(Scenario* scs) {
  const Scenario s = scs[0];
  const int m = blockIdx.x * 256 + threadIdx.x;
  if (m >= s.M) return;
  const int pos = atomicAdd(&s.vcur[s.mv[m]], 1);
  s.scratch[pos] = m;
}

// Block = (chunk c of a vehicle's missions, 512 consecutive bases): thread
// per pair of bases, eight mission rows loaded before any is accumulated.
__global__ void __launch_bounds__(256) rows_stream_kernel(Scenario* scs) {
  constexpr int NT = 256, R = 2, U = 8;
  const Scenario s = scs[0];
  const int c = blockIdx.x;
  if (c >= s.vseg[s.V + 1]) return;
  const int v = s.vch[3 * c], k0 = s.vch[3 * c + 1], n = s.vch[3 * c + 2] - k0;
  const int B = s.B;
  const int tb = blockIdx.y * (NT * R) + threadIdx.x;
  __shared__ int mk[kRowsChunk];
  __shared__ double mck[kRowsChunk];
  for (int k = threadIdx.x; k < n; k += NT) {
    const int m = s.scratch[k0 + k];
    mk[k] = m;
    mck[k] = s.mc[m];
  }
  __syncthreads();
  if (blockIdx.y * (NT * R) >= B) return;
  double as[R], aa[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    as[i] = 0.0;
    aa[i] = 0.0;
  }
  bool ok[R];
#pragma unroll
  for (int i = 0; i < R; ++i) ok[i] = tb + i * NT < B;
  int k = 0;
  for (; k + U <= n; k += U) {
    double x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* row = s.costT + (long long)mk[k + u] * B + tb;
#pragma unroll
      for (int i = 0; i < R; ++i) x[u][i] = ok[i] ? row[i * NT] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double mcm = mck[k + u];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double d = x[u][i] - mcm;
        as[i] += d;
        aa[i] += fabs(d);
      }
    }
  }
  for (; k < n; ++k) {
    const double* row = s.costT + (long long)mk[k] * B + tb;
    const double mcm = mck[k];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double d = (ok[i] ? row[i * NT] : 0.0) - mcm;
      as[i] += d;
      aa[i] += fabs(d);
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = tb + i * NT;
    if (ok[i] && s.bveh[t] < 0) {
      atomicAdd(&s.rA[tix(s, t, v)], as[i]);
      atomicAdd(&s.rU[tix(s, t, v)], aa[i]);
    }
  }
}

// Bounds and classes of the streamed rows: entry (t, v), t fastest.
__global__ void __launch_bounds__(256) rows_finish_kernel(Scenario* scs) {
  const Scenario s = scs[0];
  __shared__ Shared sh;
  if (threadIdx.x == 0) sh.c = *s.ctr;
  __syncthreads();
  const long long e = (long long)blockIdx.x * 256 + threadIdx.x;
  if (e >= (long long)s.B * s.V) return;
  const int v = (int)(e / s.B), t = (int)(e % s.B);
  if (s.bveh[t] >= 0) return;
  const int n = s.vcount[v];
  const double U = s.rU[e] * (1.0 + (double)(n + 2) * kTwoPowM52);
  s.rU[e] = U;
  s.rE[e] = (double)(n + 2) * kTwoPowM52 * U;
  if (table_class(s, sh, t, v) != CLS_POS) atomicAdd(&s.rcnt[t], 1);
}

// Exact fixed-order final total (st.total after the last move): the cached
// exact total when it is current, else one block-parallel exact chain.
__global__ void __launch_bounds__(512) final_kernel(Scenario* scs) {
  const Scenario s = scs[blockIdx.x];
  __shared__ Shared sh;
  const Counters c = *s.ctr;
  if (c.total_ver == (long long)c.applied) {
    if (threadIdx.x == 0) s.ctr->final_total = c.total_exact;
    return;
  }
  const double t = exact_chain<512>(s, sh, 0, -1, 0.0, -1, nullptr);
  if (threadIdx.x == 0) s.ctr->final_total = t;
}

// A batch's results side by side (one device-to-host copy instead of two per
// scenario): mv of scenario s at out_mv + s*M, vbase at out_vb + vb_off[s].
__global__ void __launch_bounds__(256) gather_results_kernel(const Scenario* scs, int M,
                                                             int32_t* __restrict__ out_mv,
                                                             int32_t* __restrict__ out_vb,
                                                             const long long* __restrict__ vb_off) {
  const Scenario& s = scs[blockIdx.y];
  int32_t* mv = out_mv + (long long)blockIdx.y * M;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) mv[m] = s.mv[m];
  if (blockIdx.x == 0)
    for (int v = threadIdx.x; v < s.V; v += blockDim.x) out_vb[vb_off[blockIdx.y] + v] = s.vbase[v];
}

cudaError_t launch_gather_results(const Scenario* d_scs, int n_scn, int M, int32_t* out_mv,
                                  int32_t* out_vb, const long long* vb_off, cudaStream_t stream) {
  if (n_scn <= 0) return cudaSuccess;
  gather_results_kernel<<<dim3(std::max(1, std::min((M + 255) / 256, 8)), n_scn), 256, 0, stream>>>(
      d_scs, M, out_mv, out_vb, vb_off);
  return cudaGetLastError();
}

// Host-side launch attributes, cached per kernel: a single scenario's search
// enqueues a pass per host round trip, and the attribute / occupancy queries
// were part of that latency.
namespace {
std::mutex g_attr_mu;
std::unordered_map<const void*, int> g_smem_set;                 // max dynamic smem set
std::unordered_map<const void*, std::pair<size_t, int>> g_occ;   // (smem, blocks per SM)
int g_sms = 0;

void set_smem(const void* kern, size_t smem) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_smem_set.find(kern);
  if (it != g_smem_set.end() && it->second >= (int)smem) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  g_smem_set[kern] = (int)smem;
}

int blocks_per_sm(const void* kern, int nt, size_t smem, int* sms) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  *sms = g_sms;
  auto it = g_occ.find(kern);
  if (it != g_occ.end() && it->second.first == smem) return it->second.second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem);
  g_occ[kern] = {smem, per_sm};
  return per_sm;
}
}  // namespace

template <int NT>
static cudaError_t launch_pass_nt(Scenario* d_scs, const int32_t* d_active, int n_scn,
                                  const int32_t* d_perms, int kpasses, bool inkernel,
                                  int max_passes, int M, bool tabu, long long tenure, bool debug,
                                  int V, int B, int K, int helpers_req, unsigned epoch,
                                  const int* perm_bad, cudaStream_t stream, bool global_bits) {
  const size_t core = pass_smem_core(V, NT);
  const size_t state = pass_smem_state(V, B, K);
  const size_t bits = 2 * align16(4ull * V * ((M + 31) / 32));
  const size_t limit = 220 * 1024;
  // 256-thread blocks run two per SM, 128-thread blocks four: the bitsets
  // (and mission mirrors) only join while that many fit
  size_t bits_limit = NT == 256 ? 100 * 1024 : (NT == 128 ? 54 * 1024 : limit);
  if (const char* e = std::getenv("FLEETPLACE_SMEM_KB")) bits_limit = (size_t)std::atoi(e) * 1024;
  if (core > limit) return cudaErrorInvalidConfiguration;
  const int in_smem = core + state <= limit ? 1 : 0;
  int bits_smem = in_smem && core + state + bits <= bits_limit && !global_bits ? 1 : 0;
  if (const char* e = std::getenv("FLEETPLACE_BITS_SMEM")) bits_smem = bits_smem && std::atoi(e) != 0;
  // the mission mirrors join when the bitsets did (pool bound: B + 2V + 1)
  const size_t mirrors = 2 * align16(4ull * M) + 2 * align16(4ull * (B + 2 * V + 1)) + align16(4ull * B);
  // (also without the bitsets: helper-block launches keep those in global
  // memory, the mission mirrors still fit)
  int mirrors_smem = in_smem && core + state + (bits_smem ? bits : 0) + mirrors <= bits_limit ? 1 : 0;
  if (const char* e = std::getenv("FLEETPLACE_MIRRORS_SMEM"))
    mirrors_smem = mirrors_smem && std::atoi(e) != 0;
  const size_t smem = core + (in_smem ? state : 0) + (bits_smem ? bits : 0) +
                      (mirrors_smem ? mirrors : 0);
  // HELP: the variant that can share work with helper blocks (large single
  // scenarios); the others compile none of that code
  const bool help_possible = helpers_req != 0 && n_scn == 1 && kpasses == 1 && !inkernel && !bits_smem;
  auto kern = inkernel ? pass_kernel<NT, true, false>
                       : (help_possible ? pass_kernel<NT, false, true> : pass_kernel<NT, false, false>);
  set_smem((const void*)kern, smem);
  // helper blocks: one scenario, one pass per launch, bitsets in global
  // memory, and every block co-resident (cooperative launch)
  int helpers = 0;
  if (helpers_req != 0 && n_scn == 1 && kpasses == 1 && !inkernel && !bits_smem) {
    int sms = 0;
    const int per_sm = blocks_per_sm((const void*)kern, NT, smem, &sms);
    helpers = per_sm * sms - 1;
    if (helpers_req > 0 && helpers_req < helpers) helpers = helpers_req;
    if (helpers < 0) helpers = 0;
  }
  if (helpers > 0) {
    int ip = inkernel ? 1 : 0, t = tabu ? 1 : 0, d = debug ? 1 : 0;
    void* args[] = {&d_scs, &d_active, &d_perms, &kpasses, &ip, &max_passes, &t, &tenure, &d,
                    (void*)&in_smem, (void*)&bits_smem, (void*)&mirrors_smem, &helpers, &epoch,
                    (void*)&perm_bad};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(1 + helpers),
                                                      dim3(NT), args, smem, stream);
    if (e == cudaSuccess) return e;
    // the blocks could not all be resident (another tenant, MPS limits): the
    // same pass without helpers, which is only an execution strategy
    cudaGetLastError();
    kern = pass_kernel<NT, false, false>;
    set_smem((const void*)kern, smem);
  }
  kern<<<n_scn, NT, smem, stream>>>(d_scs, d_active, d_perms, kpasses, inkernel,
                                               max_passes, tabu, tenure, debug, in_smem,
                                               bits_smem, mirrors_smem, 0, epoch, perm_bad);
  return cudaGetLastError();
}

// The grid-wide per-pass sweep (mirrors + imp/mem bitsets) for the pass whose
// permutations start at d_perms.
cudaError_t launch_sweep(Scenario* d_scs, const int32_t* d_active, int n_scn,
                         const int32_t* d_perms, int M, cudaStream_t stream) {
  const int nwd = (M + 31) / 32;
  dim3 mg((nwd + 7) / 8 < 1184 ? (nwd + 7) / 8 : 1184, n_scn);
  if (M > 0) prep_kernel<<<mg, 256, 0, stream>>>(d_scs, d_active, d_perms + M);
  return cudaGetLastError();
}

// `kpasses` passes whose permutations are consecutive in d_perms (perm_a,
// perm_b per pass). inkernel: each block rebuilds its own mirrors/bitsets
// between passes; otherwise kpasses must be 1 and the grid-wide sweep runs
// first (launch_sweep).
cudaError_t launch_pass(Scenario* d_scs, const int32_t* d_active, int n_scn,
                        const int32_t* d_perms, int kpasses, bool inkernel, int max_passes, int M,
                        bool tabu, long long tenure, bool debug, int V, int B, int K,
                        cudaStream_t stream, int threads, int helpers_req, unsigned epoch,
                        const int* perm_bad, bool global_bits) {
  if (threads == 1024)
    return launch_pass_nt<1024>(d_scs, d_active, n_scn, d_perms, kpasses, inkernel, max_passes,
                                M, tabu, tenure, debug, V, B, K, helpers_req, epoch, perm_bad, stream,
                                global_bits);
  if (threads == 128)
    return launch_pass_nt<128>(d_scs, d_active, n_scn, d_perms, kpasses, inkernel, max_passes,
                               M, tabu, tenure, debug, V, B, K, helpers_req, epoch, perm_bad, stream,
                               global_bits);
  if (threads == 512)
    return launch_pass_nt<512>(d_scs, d_active, n_scn, d_perms, kpasses, inkernel, max_passes,
                               M, tabu, tenure, debug, V, B, K, helpers_req, epoch, perm_bad, stream,
                               global_bits);
  return launch_pass_nt<256>(d_scs, d_active, n_scn, d_perms, kpasses, inkernel, max_passes,
                             M, tabu, tenure, debug, V, B, K, helpers_req, epoch, perm_bad, stream,
                             global_bits);
}

// ev[0..4]: events recorded around the four stages (may be null).
// side: a second stream, used only by the FLEETPLACE_INIT_SIDE fault probe
// (1: the exact start total concurrent with the row builds, 2: on the side
// stream but joined at once); the shipped path runs everything in order.
cudaError_t launch_init(Scenario* d_scs, const Scenario* h_scs, int n_scn, int M, int maxB,
                        int maxV, bool transpose, cudaStream_t stream, cudaEvent_t* ev,
                        bool exact_total, cudaStream_t side) {
  if (ev) cudaEventRecord(ev[0], stream);
  if (transpose && M > 0 && maxB > 0)
    transpose_kernel<<<dim3((M + 63) / 64, (maxB + 31) / 32, n_scn), 256, 0, stream>>>(d_scs);
  if (ev) cudaEventRecord(ev[1], stream);
  if (M > 0)
    mission_cost_kernel<<<dim3(std::min((M + 255) / 256, 4 * 148), n_scn), 256, 0, stream>>>(d_scs);
  const char* probe = std::getenv("FLEETPLACE_INIT_SIDE");
  const int side_mode = probe && side && side != stream && exact_total ? std::atoi(probe) : 0;
  cudaEvent_t costs_done = nullptr, total_done = nullptr;
  if (side_mode) {
    cudaEventCreateWithFlags(&costs_done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&total_done, cudaEventDisableTiming);
    cudaEventRecord(costs_done, stream);
    cudaStreamWaitEvent(side, costs_done, 0);
    init_kernel<<<n_scn, 512, 0, side>>>(d_scs);
    cudaEventRecord(total_done, side);
    if (side_mode == 2) cudaStreamWaitEvent(stream, total_done, 0);
  } else if (exact_total) {
    init_kernel<<<n_scn, 512, 0, stream>>>(d_scs);
  }
  if (ev) cudaEventRecord(ev[2], stream);
  if (M > 0) impt_init_kernel<<<dim3((M + 255) / 256, n_scn), 256, 0, stream>>>(d_scs);
  if (ev) cudaEventRecord(ev[3], stream);
  const Scenario& h = h_scs[0];
  if (n_scn == 1 && h.costT && M > 0 && maxB > 0 && maxV > 0) {
    // single scenario with the row-major copy: stream it by vehicle chunks
    const size_t bv = (size_t)h.B * h.V;
    cudaMemsetAsync(h.rA, 0, sizeof(double) * bv, stream);
    cudaMemsetAsync(h.rU, 0, sizeof(double) * bv, stream);
    cudaMemsetAsync(h.rcnt, 0, sizeof(int32_t) * h.B, stream);
    rows_plan_kernel<<<1, 32, 0, stream>>>(d_scs);
    rows_group_kernel<<<(M + 255) / 256, 256, 0, stream>>>(d_scs);
    const int chunks = M / kRowsChunk + maxV + 1;
    rows_stream_kernel<<<dim3(chunks, (maxB + 511) / 512), 256, 0, stream>>>(d_scs);
    rows_finish_kernel<<<(unsigned)((bv + 255) / 256), 256, 0, stream>>>(d_scs);
  } else {
    const size_t smem = sizeof(double) * (16ull * maxV + 8 * 32);
    cudaFuncSetAttribute(table_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (maxB > 0) table_rows_kernel<<<dim3(maxB, n_scn), 256, smem, stream>>>(d_scs);
  }
  if (side_mode) {
    cudaStreamWaitEvent(stream, total_done, 0);
    cudaEventDestroy(total_done);
    cudaEventDestroy(costs_done);
  }
  if (ev) cudaEventRecord(ev[4], stream);
  return cudaGetLastError();
}

cudaError_t launch_final(Scenario* d_scs, int n_scn, cudaStream_t stream) {
  final_kernel<<<n_scn, 512, 0, stream>>>(d_scs);
  return cudaGetLastError();
}

}  // namespace fpk
