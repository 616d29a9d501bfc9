// common.cuh — device-side types shared by the fleetplace_b200 kernels.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace fpk {

// Tabu roles (proj/include/fleetplace/search.hpp:78-79).
enum : uint8_t { ROLE_OUTER = 0, ROLE_INNER = 1 };
// Pool entry kinds (proj/include/fleetplace/search.hpp:30-32).
enum : int32_t { POOL_EMPTY = 0, POOL_IDLE = 1 };

// Per-scenario counters and block-uniform scalars of the search automaton.
// Lives in device memory between pass launches; the pass kernel keeps a copy
// in shared memory and writes it back on exit.
struct Counters {
  long long tick;                 // pairs visited so far (tabu clock)
  unsigned long long evaluations;
  unsigned long long applied;
  unsigned long long skips_outer;
  unsigned long long skips_inner;
  unsigned long long fallbacks;   // accept decisions settled by exact chains
  long long passes;               // passes completed
  int done;                       // search finished (quiescent, max_passes or error)
  int psize;                      // current pool size
  int pass_applied;               // moves applied in the current pass
  int pass_relocs;                // relocations applied in the current pass
  int pass_skipped;               // any tabu skip in the current pass
  int error;                      // 0 = ok, else an fp_status
  int force_exact;                // test hook: 1 = every total comparison through the exact
                                  // chains, 2 = every unsettled relocation delta exactly
  int chain_mode;                 // 0 = helper-assisted exact chains when possible, 1 = never
  int hp_valid;                   // chunk boundaries [0, hp_valid] of hP hold the current state's
                                  //   exact running sums (helper-assisted chains)
  int check_impt;                 // test hook: verify impT against the table every pass
  double total_up;                // rigorous upper bound of the current total
  double final_total;             // exact fixed-order total (written at the end)
  double total_exact;             // exact fixed-order total of the state ...
  long long total_ver;            // ... at this applied-move count (-1: unknown)
  // SM cycles spent per automaton phase (thread 0's view): 0 row runs,
  // 1 row contexts, 2 scan steps, 3 event pairs, 4 exact fallbacks, 5 exact
  // table-row rebuilds, 6 relocation bit updates, 7 substitution bit
  // updates, 8 relocation apply, 9 exact totals, 10 table patches, 11
  // per-pass setup, 12 exact relocation deltas, 13 exact candidate totals,
  // 14 helper waits, 15 reserved
  unsigned long long cycles[16];
  // event counts: 0 scanned rows, 1 scan steps, 2 row contexts, 3 exact
  // table-row rebuilds, 4 rows resolved by the O(1) eventless test
  unsigned long long counts[5];
};

// Work sharing for large single scenarios: the pass kernel runs one master
// block (the automaton) plus helper blocks that split the O(M) work of a
// relocation. The master posts a job by publishing seq = (epoch << 32) | k
// (epoch = launch number, k = job number within the launch); every helper
// adds one to `done` when its share is finished.
enum : int { HJOB_QUIT = 0, HJOB_RELOCATE = 1, HJOB_CHAIN = 2, HJOB_LOG = 3 };

// A reassignment / takeover for the relocation-delta table, applied by the
// helper blocks in the background (each helper owns a slice of the bases).
struct SubRec {
  int j, loser, gain, nl, ng, pad;
  double mc_old, mc_new;
};
constexpr int kLogCap = 1024;
struct HelperCtl {
  unsigned long long seq;
  unsigned done;
  int kind;
  int x, t, b_old;   // relocation: mover, target base, vacated base
  int impc_x;        // out: set bits of the mover's new imp row
  int ckind, cj, cmover, ct;  // chain: term kind, mission, mover, base (-1)
  double cnewc;               // chain: the substituted cost (kind 1)
  int cstart;                 // chain: first chunk
  int minm;                   // relocation: smallest mission index of the mover
  unsigned long long log_tail;  // (launch << 32) | records published in the launch
  unsigned log_done;            // helper-record completions, cumulative
};

// Exact fixed-order sums are walked in chunks of kChainSub terms (see
// exact_chain_helped).
constexpr int kChainSub = 2048;
// Missions per block of the row-major relocation-table build.
constexpr int kRowsChunk = 256;
constexpr int kNoBinade = -100000;

// std::mt19937_64 state (the search's permutation stream, perm_kernels.cu).
// One scenario's table build in a batched kernel (1) launch.
struct TableJob {
  const double *blat, *blon, *bcos, *plat, *plon, *pcos, *dlat, *dlon, *dcos;
  double* cost;
  int B;
};

struct MtState {
  unsigned long long mt[312];
  int idx;
};

// Up to kMax seeds passed by value to mt_seed_kernel (no host copy).
struct MtSeeds {
  static constexpr int kMax = 64;
  unsigned long long seed[kMax];
};

// One search scenario: the resident distance table plus the index-based
// SearchState of proj/src/search_state.hpp:20-31 in structure-of-arrays
// form, the perm_b-ordered mirrors the scan streams, and the expiry-stamp
// tabu table.
struct Scenario {
  // read-only instance data
  const double* cost;        // [B*M] column-major, entry (m, b) at b*M + m
  const double* costT;       // [M*B] row-major copy, entry (m, b) at m*B + b, or null
  const uint8_t* ro;         // [M] mission rotary_only
  const uint8_t* vfixed;     // [V] vehicle is fixed-wing
  const uint8_t* bheli;      // [B] base is a helipad
  const int32_t* vrk;        // [V] slot of {Relocate, vehicle id} key
  const int32_t* brk;        // [B] slot of {Relocate, base id} key
  // mutable state (natural mission order)
  int32_t* mv;               // [M] mission -> vehicle index
  double* mc;                // [M] cost charged per mission
  int32_t* vbase;            // [V] vehicle -> base index (-1 unplaced)
  int32_t* vcount;           // [V] missions per vehicle
  int32_t* bveh;             // [B] base -> vehicle index or -1
  int32_t* pkind;            // [pool_cap]
  int32_t* pidx;             // [pool_cap] base index or vehicle index
  // perm_b-ordered mirrors, rebuilt per pass
  int32_t* mvp;              // [M] mv[perm_b[p]]
  double* mcp;               // [M] mc[perm_b[p]]
  uint8_t* rop;              // [M] ro[perm_b[p]]
  int32_t* invb;             // [M] position of mission m in perm_b
  // tabu: expiry stamps; takeover/reassign keys are only ever Outer
  long long* exp_take;       // [V] {Takeover, vehicle id}
  long long* exp_reas;       // [V] {Reassign, vehicle id}
  long long* exp_rel;        // [K] {Relocate, id}, ids of bases and vehicles
  uint8_t* role_rel;         // [K]
  // relocation-delta table, entry (t, v) at v*B + t, t an empty base, v a
  // vehicle:
  //  rA ~ X = sum over v's missions of (cost(m, t) - mc[m]) (exact reals),
  //  |rA - X| <= rE, rU >= sum |cost(m, t) - mc[m]|; rcnt[t] = vehicles whose
  //  relocation to t is not certainly non-improving
  double* rA;                // [B*V]
  double* rE;                // [B*V]
  double* rU;                // [B*V]
  int32_t* rcnt;             // [B]
  // perm_b-position bitsets, word w covers positions [32w, 32w+32):
  //  imp[g]: reassigning / taking over that position's mission to vehicle g
  //          would lower its cost (mv != g, compatible, cost(j, base(g)) < mc[j])
  //  mem[v]: the position's mission is served by vehicle v
  uint32_t* imp;             // [V*NWD]
  uint32_t* mem;             // [V*NWD]
  // the same improvement bits in natural mission order, one row of NVW words
  // per mission (bit g of row j: moving mission j to vehicle g lowers its
  // cost); maintained on every move, so the per-pass rebuild of imp is a
  // gather of M rows instead of V*M table entries
  uint32_t* impT;            // [M*NVW]
  // relocation-table build from the row-major copy: missions grouped by
  // vehicle (in scratch), per-vehicle segment starts / cursors, chunk plan
  int32_t* vseg;             // [V+2] segment starts, [V] = M, [V+1] = chunk count
  int32_t* vcur;             // [V]
  int32_t* vch;              // [3*(M/kRowsChunk + V + 1)] (vehicle, begin, end)
  int32_t* scratch;          // [M] per-scenario scratch (relocation position lists)
  HelperCtl* hc;             // helper work sharing (zeroed at search start)
  int32_t* hdelta;           // [V] helpers' imp-row popcount deltas
  double* hsum;              // [V] helpers' partial relocation sums (fresh row)
  double* habs;              // [V]
  int32_t* hec;              // [ceil(M/kChainSub)] binade of the running sum at each chunk
                             //   start in the latest exact chain (kNoBinade: unknown)
  long long* hrs;            // [..] helpers: chunk sums of rn(term / ulp) in binade hue
  SubRec* hlog;              // [kLogCap] substitution records for the helpers
  double* hP;                // [nsub+1] exact running sum at each chunk start (current state)
  double* hP2;               // [nsub+1] the same for the last candidate chain (adopted if accepted)
  int32_t* hue;              // [..] helpers: the binade hrs is for, kNoBinade when the
                             //   chunk holds a rounding tie / a huge term / no prediction
  Counters* ctr;
  int32_t M, B, V, K, pool_cap, nwd, nvw;
  // per-scenario SearchConfig (a batch may mix seeds, modes, tenures and
  // pass caps: run_experiment's attempts, proj/src/bench.cpp:125-128)
  long long tenure;          // resolved tabu tenure (0 in local mode)
  int32_t max_passes;        // < 0: no cap
  int32_t tabu;              // 1 = tabu_search, 0 = local_search
  int32_t debug;             // debug_check_deltas
  int32_t pstream;           // index of this scenario's permutation stream in a chunk
};

}  // namespace fpk

#define FP_CUDA_CHECK(expr)                                                \
  do {                                                                     \
    cudaError_t err__ = (expr);                                            \
    if (err__ != cudaSuccess) throw ::fpk_host::CudaError(err__, #expr);   \
  } while (0)
