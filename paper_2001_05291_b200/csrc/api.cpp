// api.cpp — the C ABI (include/fleetplace_b200.h): validation, host-side
// selection logic, device memory and the search orchestration around the
// kernels in table_rank_kernels.cu and search_kernels.cu.
//
// Host logic kept here is the reference's O(B log B) / O(V) bookkeeping
// (sorting bases, helipad cap, placement order, pool construction, input
// validation) and the sequential mt19937_64 permutation stream; everything
// that touches the M x B table runs on the device.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "host_common.hpp"

namespace fpk_host {
void generate_instance(uint64_t pool_seed, const double* bbox, int aerodromes, int helipads,
                       int health_sites, int missions, double rotary_only_fraction,
                       uint64_t seed, int rotary, int fixed_wing, int32_t* base_id,
                       uint8_t* base_kind, double* base_lat, double* base_lon,
                       int32_t* vehicle_id, uint8_t* vehicle_kind, int32_t* mission_id,
                       double* pickup_lat, double* pickup_lon, double* delivery_lat,
                       double* delivery_lon, uint8_t* rotary_only);
}

using fpk_host::CudaError;
using fpk_host::FpError;

struct fp_ctx {
  int device = 0;
  bool row_copy = true;  // eager row-major copy after build / upload (fp_ctx_set_row_copy)
  cudaStream_t stream = nullptr;
  double* d_cost = nullptr;
  size_t cost_cap = 0;  // elements
  int M = -1, B = -1;
  // every entry of the resident table is finite and >= 0 (kernel (1) tables
  // are by construction; uploads are checked): the search's exact-sum
  // machinery relies on it
  bool table_ok = false;
  int* d_flag = nullptr;  // device word for the table check (allocated once)
  // pinned host staging (grow-only): search region A, batch point coordinates
  unsigned char* h_stage = nullptr;
  size_t h_stage_cap = 0;
  double* h_pts = nullptr;
  size_t h_pts_cap = 0;
  // pinned per-chunk control words of a search (counters, active flags, the
  // rejected-draw flag): pageable copies would stage through the driver
  unsigned char* h_small = nullptr;
  size_t h_small_cap = 0;
  uint64_t launches = 0;
  double last_kernel_ms = 0.0;
  // pinned staging for permutations (double-buffered)
  int32_t* h_perm[2] = {nullptr, nullptr};
  size_t perm_cap = 0;
  // device workspace of the searches (grow-only: no allocation per call)
  unsigned char* ws = nullptr;
  size_t ws_cap = 0;
  // row-major copy of the resident table, made on a second stream as soon
  // as the table is resident (overlapping ranking), reused by every search
  double* d_costT = nullptr;
  size_t costT_cap = 0;   // elements
  bool costT_valid = false;
  cudaStream_t aux = nullptr;
  cudaStream_t pstream = nullptr;  // a batch's first permutation draws (overlap its start)
  cudaEvent_t table_ready = nullptr, costT_ready = nullptr;
  cudaEvent_t copy_t0 = nullptr, copy_t1 = nullptr;  // timing of the copy
  bool copy_timed = false;
};

namespace {

thread_local std::string g_err;

fp_status fail(fp_status c, const std::string& m) {
  g_err = m;
  return c;
}

template <typename F>
fp_status guarded(F&& f) {
  try {
    f();
    return FP_OK;
  } catch (const FpError& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(FP_ERR_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(FP_ERR_ERROR, e.what());
  }
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(e, what);
}

// RAII device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  // with a stream: stream-ordered (cudaMallocAsync / cudaFreeAsync), so the
  // free does not wait for the whole device (e.g. the row-major table copy
  // running on the context's second stream)
  cudaStream_t s = nullptr;
  DBuf() = default;
  explicit DBuf(size_t count, cudaStream_t st = nullptr) : s(st) { alloc(count); }
  void alloc(size_t count) {
    free_();
    n = count;
    if (count) {
      if (s) check(cudaMallocAsync(&p, sizeof(T) * count, s), "cudaMallocAsync");
      else check(cudaMalloc(&p, sizeof(T) * count), "cudaMalloc");
    }
  }
  void free_() {
    if (p) {
      if (s) cudaFreeAsync(p, s);
      else cudaFree(p);
    }
    p = nullptr;
  }
  ~DBuf() { free_(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      free_();
      p = o.p;
      n = o.n;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
};

template <typename T>
void h2d(T* d, const T* h, size_t n, cudaStream_t st) {
  if (n) check(cudaMemcpyAsync(d, h, sizeof(T) * n, cudaMemcpyHostToDevice, st), "H2D");
}
template <typename T>
void d2h(T* h, const T* d, size_t n, cudaStream_t st) {
  if (n) check(cudaMemcpyAsync(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost, st), "D2H");
}

// Waits for the stream. blocking: the thread sleeps on a blocking-sync event
// instead of spinning -- for the long waits of batch launches (hundreds of
// ms), where a spinning thread burns the process's CPU quota and a quota-
// throttled process wakes tens of ms late; short waits spin (lower latency).
void wait_stream(cudaStream_t st, bool blocking, const char* what) {
  if (!blocking) {
    check(cudaStreamSynchronize(st), what);
    return;
  }
  cudaEvent_t e;
  check(cudaEventCreateWithFlags(&e, cudaEventBlockingSync | cudaEventDisableTiming), what);
  cudaError_t r = cudaEventRecord(e, st);
  if (r == cudaSuccess) r = cudaEventSynchronize(e);
  cudaEventDestroy(e);
  check(r, what);
}

void ensure_table(const fp_ctx* ctx, int M, int B) {
  if (ctx->M != M || ctx->B != B || (size_t)M * B > 0 && !ctx->d_cost)
    throw FpError(FP_ERR_INVALID_ARGUMENT,
                  "no resident distance table of shape " + std::to_string(M) + "x" +
                      std::to_string(B) + " (call fp_build_distance_table or fp_table_upload)");
}

void table_alloc(fp_ctx* ctx, int M, int B) {
  if (ctx->aux) cudaStreamSynchronize(ctx->aux);  // a pending copy still reads the table
  const size_t need = (size_t)M * (size_t)B;
  if (need > ctx->cost_cap) {
    if (ctx->d_cost) cudaFree(ctx->d_cost);
    ctx->d_cost = nullptr;
    ctx->cost_cap = 0;
    // +2 doubles: 16-byte tail padding for the aligned bulk copies of kernel (2)
    check(cudaMalloc(&ctx->d_cost, sizeof(double) * (need + 2)), "cudaMalloc(table)");
    ctx->cost_cap = need;
  }
  ctx->M = M;
  ctx->B = B;
  ctx->costT_valid = false;
  ctx->table_ok = false;
}

// fn(0..n-1) on up to 16 host threads (per-scenario host work of batches);
// the first exception is rethrown.
template <typename Fn>
void parallel_for(int n, Fn&& fn, int min_n = 64) {
  const int T = std::min(n, (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 16u));
  if (n < min_n || T <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> ws;
  std::vector<std::exception_ptr> errs(T);
  for (int t = 0; t < T; ++t)
    ws.emplace_back([&, t] {
      try {
        for (int i = (int)((long long)n * t / T); i < (int)((long long)n * (t + 1) / T); ++i) fn(i);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& w : ws) w.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

bool valid_point(double lat, double lon) {
  return lat >= -90.0 && lat <= 90.0 && lon >= -180.0 && lon <= 180.0;
}

// The missions' checks of validate_instance on host threads: ids unique
// (a bitmap over a compact id range, set with atomic ors) and coordinates in
// range (branch-free, vectorised). true = every mission passes; false =
// some mission fails, or the ids are not compact -- the sequential scan then
// runs and reports the first failure in load order. c4 (1M missions):
// ~8 ms sequential.
bool missions_ok_fast(const fp_instance* in) {
  const int M = in->n_missions;
  if (M < (1 << 16)) return false;  // small: the sequential scan is cheap
  constexpr int kParts = 64;
  int los[kParts], his[kParts];
  parallel_for(kParts, [&](int t) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int m = (int)((long long)M * t / kParts); m < (int)((long long)M * (t + 1) / kParts); ++m) {
      lo = std::min(lo, in->mission_id[m]);
      hi = std::max(hi, in->mission_id[m]);
    }
    los[t] = lo;
    his[t] = hi;
  });
  const int lo = *std::min_element(los, los + kParts), hi = *std::max_element(his, his + kParts);
  const int64_t span = (int64_t)hi - lo + 1;
  if (span > 8 * (int64_t)M + 4096) return false;
  std::vector<uint64_t> bits((size_t)((span + 63) / 64), 0);
  std::atomic<int> bad{0};
  parallel_for(kParts, [&](int t) {
    int ok = 1;
    const int m0 = (int)((long long)M * t / kParts), m1 = (int)((long long)M * (t + 1) / kParts);
    for (int m = m0; m < m1; ++m) {
      const double a = in->pickup_lat[m], b = in->pickup_lon[m];
      const double c = in->delivery_lat[m], d = in->delivery_lon[m];
      ok &= (a >= -90.0) & (a <= 90.0) & (b >= -180.0) & (b <= 180.0) & (c >= -90.0) &
            (c <= 90.0) & (d >= -180.0) & (d <= 180.0);
    }
    for (int m = m0; m < m1 && ok; ++m) {
      const uint64_t k = (uint64_t)((int64_t)in->mission_id[m] - lo);
      const uint64_t bit = 1ull << (k & 63);
      if (__atomic_fetch_or(&bits[k >> 6], bit, __ATOMIC_RELAXED) & bit) ok = 0;
    }
    if (!ok) bad.store(1, std::memory_order_relaxed);
  });
  return bad.load() == 0;
}

// validate_instance, proj/src/model.cpp:46-74 (same checks, same order).
void validate(const fp_instance* in) {
  if (in->n_vehicles <= 0) throw FpError(FP_ERR_VALIDATION, "validation failed for fleet: must not be empty");
  if (in->n_bases <= 0) throw FpError(FP_ERR_VALIDATION, "validation failed for bases: must not be empty");
  {
    std::unordered_map<int, int> seen;
    seen.reserve(in->n_bases * 2);
    for (int b = 0; b < in->n_bases; ++b) {
      if (!seen.emplace(in->base_id[b], b).second)
        throw FpError(FP_ERR_VALIDATION, "validation failed for base " +
                                             std::to_string(in->base_id[b]) + ": duplicate id");
      if (!valid_point(in->base_lat[b], in->base_lon[b]))
        throw FpError(FP_ERR_VALIDATION, "validation failed for base " +
                                             std::to_string(in->base_id[b]) +
                                             ": coordinates out of range");
    }
  }
  {
    std::unordered_map<int, int> seen;
    for (int v = 0; v < in->n_vehicles; ++v)
      if (!seen.emplace(in->vehicle_id[v], v).second)
        throw FpError(FP_ERR_VALIDATION, "validation failed for vehicle " +
                                             std::to_string(in->vehicle_id[v]) + ": duplicate id");
  }
  if (!missions_ok_fast(in)) {
    // the first failing mission in load order (the reference's error): a
    // bitmap over the id range when it is compact (generated ids are dense,
    // proj/src/data.cpp:156-174), else a map
    const int M = in->n_missions;
    int lo = INT_MAX, hi = INT_MIN;
    for (int m = 0; m < M; ++m) {
      lo = std::min(lo, in->mission_id[m]);
      hi = std::max(hi, in->mission_id[m]);
    }
    const int64_t span = M ? (int64_t)hi - lo + 1 : 0;
    std::vector<uint64_t> bits(span <= 8 * (int64_t)M + 4096 ? (size_t)((span + 63) / 64) : 0);
    std::unordered_map<int, int> seen;
    if (bits.empty()) seen.reserve((size_t)M * 2);
    for (int m = 0; m < M; ++m) {
      bool dup;
      if (!bits.empty()) {
        const uint64_t k = (uint64_t)((int64_t)in->mission_id[m] - lo);
        dup = (bits[k >> 6] >> (k & 63)) & 1;
        bits[k >> 6] |= 1ull << (k & 63);
      } else {
        dup = !seen.emplace(in->mission_id[m], m).second;
      }
      if (dup)
        throw FpError(FP_ERR_VALIDATION, "validation failed for mission " +
                                             std::to_string(in->mission_id[m]) + ": duplicate id");
      if (!valid_point(in->pickup_lat[m], in->pickup_lon[m]) ||
          !valid_point(in->delivery_lat[m], in->delivery_lon[m]))
        throw FpError(FP_ERR_VALIDATION, "validation failed for mission " +
                                             std::to_string(in->mission_id[m]) +
                                             ": coordinates out of range");
    }
  }
  int aero = 0, fixed = 0;
  for (int b = 0; b < in->n_bases; ++b) aero += in->base_kind[b] == FP_AERODROME;
  for (int v = 0; v < in->n_vehicles; ++v) fixed += in->vehicle_kind[v] == FP_FIXED;
  if (aero < fixed)
    throw FpError(FP_ERR_VALIDATION,
                  "validation failed for fleet: needs at least one aerodrome per fixed-wing vehicle");
}

// CUDA-event timer on a stream.
struct EvTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  explicit EvTimer(cudaStream_t s) : st(s) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  double stop_ms() {
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
  ~EvTimer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

// One device pass over a table: every entry finite and >= 0 (synchronises).
bool table_entries_ok(fp_ctx* ctx, const double* d_t, size_t n, cudaStream_t st) {
  if (!ctx->d_flag) check(cudaMalloc(&ctx->d_flag, sizeof(int)), "cudaMalloc(flag)");
  check(fpk::launch_table_check(d_t, n, ctx->d_flag, st), "table_check");
  ctx->launches += 1;
  int h = 0;
  d2h(&h, ctx->d_flag, 1, st);
  check(cudaStreamSynchronize(st), "table check sync");
  return h == 0;
}

// ctx->h_pts holds at least n doubles (pinned, grow-only; its previous
// contents are not kept: every user syncs before returning)
void pinned_points(fp_ctx* ctx, size_t n) {
  if (ctx->h_pts_cap >= n) return;
  if (ctx->h_pts) cudaFreeHost(ctx->h_pts);
  ctx->h_pts = nullptr;
  ctx->h_pts_cap = 0;
  check(cudaMallocHost(&ctx->h_pts, sizeof(double) * n), "pinned points");
  ctx->h_pts_cap = n;
}

// kernel (1) (build_distance_table, proj/src/model.cpp:76-90) into `dst`
// (M x B column-major) on the context's stream; ctx's resident table is
// untouched unless dst is it.
void build_table_into(fp_ctx* ctx, const fp_instance* in, double radius_km, double* dst) {
  const int M = in->n_missions, B = in->n_bases;
  cudaStream_t st = ctx->stream;
  DBuf<double> pts(6ull * M + 3ull * B, st);
  double* plat = pts.p;
  double* plon = plat + M;
  double* dlat = plon + M;
  double* dlon = dlat + M;
  double* blat = dlon + M;
  double* blon = blat + B;
  double* cosv = blon + B;  // [B + 2M]: bases, pickups, deliveries
  if ((size_t)M >= (1u << 16)) {
    // large instances: packed on host threads into the context's pinned
    // buffer, one copy (pageable copies stage through the driver: c4's 32 MB
    // of coordinates 2.5 -> ~1 ms)
    const size_t n = 4ull * M + 2ull * B;
    pinned_points(ctx, n);
    double* hp = ctx->h_pts;
    const double* src[6] = {in->pickup_lat, in->pickup_lon, in->delivery_lat, in->delivery_lon,
                            in->base_lat, in->base_lon};
    const size_t len[6] = {(size_t)M, (size_t)M, (size_t)M, (size_t)M, (size_t)B, (size_t)B};
    constexpr int kParts = 64;
    parallel_for(6 * kParts, [&](int k) {
      const int a = k / kParts, t = k % kParts;
      size_t off = 0;
      for (int q = 0; q < a; ++q) off += len[q];
      const size_t lo = len[a] * t / kParts, hi = len[a] * (t + 1) / kParts;
      std::memcpy(hp + off + lo, src[a] + lo, sizeof(double) * (hi - lo));
    });
    h2d(plat, hp, n, st);  // plat .. blon are contiguous in the same order
  } else {
    h2d(plat, in->pickup_lat, M, st);
    h2d(plon, in->pickup_lon, M, st);
    h2d(dlat, in->delivery_lat, M, st);
    h2d(dlon, in->delivery_lon, M, st);
    h2d(blat, in->base_lat, B, st);
    h2d(blon, in->base_lon, B, st);
  }
  check(fpk::launch_point_cos(blat, B, cosv, st), "cos(bases)");
  check(fpk::launch_point_cos(plat, M, cosv + B, st), "cos(pickups)");
  check(fpk::launch_point_cos(dlat, M, cosv + B + M, st), "cos(deliveries)");
  EvTimer tk(st);
  int sites = 0;
  if (std::getenv("FLEETPLACE_TRACE")) std::fprintf(stderr, "[fleetplace trace] build: points staged\n");
  check(fpk::launch_table_auto(blat, blon, cosv, B, plat, plon, cosv + B, dlat, dlon,
                               cosv + B + M, M, radius_km, dst, st, &sites),
        "table_kernel");
  ctx->last_kernel_ms = tk.stop_ms();
  ctx->launches += sites ? 10 : 4;
}

// ---- permutations (proj/include/fleetplace/rng.hpp:14-42) ------------------
struct PermStream {
  std::mt19937_64 rng;
  explicit PermStream(uint64_t seed) : rng(seed) {}
  uint64_t below(uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    uint64_t x = rng();
    while (x < threshold) x = rng();
    return x % n;
  }
  void perm(int n, int32_t* out) {
    for (int i = 0; i < n; ++i) out[i] = i;
    for (int64_t i = n; i > 1; --i) {
      const int64_t j = (int64_t)below((uint64_t)i);
      std::swap(out[i - 1], out[j]);
    }
  }
  // The same `count` permutations of n, faster for large n: the generator's
  // raw outputs first (the only sequential part), then the Fisher-Yates
  // shuffles on host threads -- permutation p consumes draws
  // [p(n-1), (p+1)(n-1)) unless a draw is rejected (x < (2^64 - i) mod i,
  // probability ~n/2^64 per draw); a rejection anywhere redoes the chunk
  // sequentially from the saved generator state, so the stream is exact.
  void perms(int n, int count, int32_t* out, std::vector<uint64_t>& raw) {
    if (n < (32 << 10) || count < 2) {
      for (int p = 0; p < count; ++p) perm(n, out + (size_t)p * n);
      return;
    }
    const std::mt19937_64 saved = rng;
    const size_t per = (size_t)n - 1;
    raw.resize(per * count);
    for (auto& x : raw) x = rng();
    std::atomic<bool> rejected{false};
    parallel_for(count, [&](int p) {
      int32_t* o = out + (size_t)p * n;
      const uint64_t* r = raw.data() + per * p;
      for (int i = 0; i < n; ++i) o[i] = i;
      for (int64_t i = n, k = 0; i > 1; --i, ++k) {
        const uint64_t x = r[k], ui = (uint64_t)i;
        if (x < ui && x < (0 - ui) % ui) {  // (the threshold is below i)
          rejected = true;
          return;
        }
        std::swap(o[i - 1], o[x % ui]);
      }
    }, 2);
    if (rejected) {
      rng = saved;
      for (int p = 0; p < count; ++p) perm(n, out + (size_t)p * n);
    }
  }
};

// ---- search setup -------------------------------------------------------------
struct HostScenario {
  const fp_instance* in;
  std::vector<int32_t> vbase, mv, vcount, bveh, pkind, pidx, vrk, brk;
  std::vector<uint8_t> vfixed, bheli;
  int K = 0;
  int psize = 0;
};

// tabu_search / local_search preconditions (proj/src/search.cpp:438-460)
// and SearchState::from (proj/src/search.cpp:14-65), index form.
HostScenario prepare(const fp_instance* in, const fp_search_start* st) {
  HostScenario h;
  h.in = in;
  const int V = in->n_vehicles, B = in->n_bases, M = in->n_missions;
  h.vbase.assign(V, -1);
  h.mv.assign(M, -1);
  h.bveh.assign(B, -1);
  h.vcount.assign(V, 0);
  // placement, iterated in vehicle-id order like std::map<int,int>
  std::vector<int> vorder(V);
  std::iota(vorder.begin(), vorder.end(), 0);
  std::sort(vorder.begin(), vorder.end(),
            [&](int a, int b) { return in->vehicle_id[a] < in->vehicle_id[b]; });
  for (int v : vorder) {
    const int b = st->vehicle_base[v];
    if (b == -1) continue;
    if (b < -1 || b >= B) throw FpError(FP_ERR_INFEASIBLE, "assignment references unknown ids");
    h.vbase[v] = b;
    h.bveh[b] = v;
  }
  for (int m = 0; m < M; ++m) {
    const int v = st->mission_vehicle[m];
    if (v == -1) continue;
    if (v < -1 || v >= V || h.vbase[v] < 0)
      throw FpError(FP_ERR_INFEASIBLE, "service references unplaced vehicle");
    h.mv[m] = v;
    h.vcount[v] += 1;
  }
  for (int m = 0; m < M; ++m)
    if (h.mv[m] < 0) throw FpError(FP_ERR_INFEASIBLE, "search start must serve every mission");
  for (int k = 0; k < st->pool_size; ++k) {
    const int x = st->pool_index[k];
    if (st->pool_kind[k] == FP_POOL_EMPTY_BASE) {
      if (x < 0 || x >= B || h.bveh[x] >= 0)
        throw FpError(FP_ERR_INFEASIBLE, "pool lists an occupied or unknown base");
      h.pkind.push_back(fpk::POOL_EMPTY);
    } else {
      if (x < 0 || x >= V || h.vcount[x] != 0)
        throw FpError(FP_ERR_INFEASIBLE, "pool lists a busy or unknown vehicle");
      h.pkind.push_back(fpk::POOL_IDLE);
    }
    h.pidx.push_back(x);
  }
  h.psize = st->pool_size;
  h.vfixed.resize(V);
  h.bheli.resize(B);
  for (int v = 0; v < V; ++v) h.vfixed[v] = in->vehicle_kind[v] == FP_FIXED;
  for (int b = 0; b < B; ++b) h.bheli[b] = in->base_kind[b] == FP_HELIPAD;
  // {Relocate, id}: base ids and vehicle ids share one key space
  // (proj/src/search.cpp:234-245, 256-263).
  std::unordered_map<int, int> slot;
  slot.reserve((size_t)(B + V) * 2);
  h.brk.resize(B);
  h.vrk.resize(V);
  for (int b = 0; b < B; ++b) h.brk[b] = slot.emplace(in->base_id[b], (int)slot.size()).first->second;
  for (int v = 0; v < V; ++v) h.vrk[v] = slot.emplace(in->vehicle_id[v], (int)slot.size()).first->second;
  h.K = (int)slot.size();
  return h;
}

long long resolve_tenure(const fp_search_config* cfg, int M) {
  if (cfg->mode != FP_MODE_TABU) return 0;
  if (cfg->tabu_tenure < 0)
    throw FpError(FP_ERR_INVALID_ARGUMENT, "tabu tenure must be positive (0 = auto)");
  const long long tenure = cfg->tabu_tenure > 0 ? cfg->tabu_tenure : 2LL * M;
  if (tenure <= 0) throw FpError(FP_ERR_INVALID_ARGUMENT, "tabu tenure must be positive");
  return tenure;
}


size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t ro, vfixed, bheli, vrk, brk, mv, mc, vbase, vcount, bveh, pkind, pidx, mvp, mcp, rop,
      invb, exp_take, exp_reas, exp_rel, role_rel, rA, rE, rU, rcnt, imp, mem, scratch, hc, hdelta,
      hsum, habs, hec, hrs, hue, impT, vseg, vcur, vch, hlog, hP, hP2, cost, totalA, totalB;
};

// Per-scenario layout in two regions: A holds what the host initialises
// (inputs, tabu stamps, zeroed control blocks; staged with one copy), B the
// device-built working arrays (never staged).
Layout layout(int M, int B, int V, int K, int cap, bool own_cost) {
  Layout L{};
  size_t a = 0, b = 0;
  auto putA = [&](size_t bytes) {
    const size_t at = a;
    a = align_up(a + bytes);
    return at;
  };
  auto putB = [&](size_t bytes) {
    const size_t at = b;
    b = align_up(b + bytes);
    return at;
  };
  L.ro = putA(M);
  L.vfixed = putA(V);
  L.bheli = putA(B);
  L.vrk = putA(4ull * V);
  L.brk = putA(4ull * B);
  L.mv = putA(4ull * M);
  L.vbase = putA(4ull * V);
  L.vcount = putA(4ull * V);
  L.bveh = putA(4ull * B);
  L.pkind = putA(4ull * cap);
  L.pidx = putA(4ull * cap);
  L.exp_take = putA(8ull * V);
  L.exp_reas = putA(8ull * V);
  L.exp_rel = putA(8ull * K);
  L.role_rel = putA(K);
  L.hc = putA(sizeof(fpk::HelperCtl));
  L.hdelta = putA(4ull * V);
  L.hsum = putA(8ull * V);
  L.habs = putA(8ull * V);
  const size_t nsub = ((size_t)M + fpk::kChainSub - 1) / fpk::kChainSub + 1;
  L.hec = putA(4ull * nsub);
  L.cost = own_cost ? putB(8ull * M * B + 16) : 0;
  L.mc = putB(8ull * M);
  L.mvp = putB(4ull * M);
  L.mcp = putB(8ull * M);
  L.rop = putB(M);
  L.invb = putB(4ull * M);
  L.rA = putB(8ull * B * V);
  L.rE = putB(8ull * B * V);
  L.rU = putB(8ull * B * V);
  L.rcnt = putB(4ull * B);
  const size_t nwd = ((size_t)M + 31) / 32;
  L.imp = putB(4ull * V * nwd);
  L.mem = putB(4ull * V * nwd);
  L.scratch = putB(4ull * M + 4);
  L.hrs = putB(8ull * nsub);
  L.hue = putB(4ull * nsub);
  L.impT = putB(4ull * M * ((V + 31) / 32) + 16);
  L.vseg = putB(4ull * (V + 2));
  L.vcur = putB(4ull * V + 4);
  L.vch = putB(12ull * ((size_t)M / fpk::kRowsChunk + V + 1));
  L.hlog = putB(sizeof(fpk::SubRec) * fpk::kLogCap);
  L.hP = putB(8ull * (nsub + 1));
  L.hP2 = putB(8ull * (nsub + 1));
  L.totalA = a;
  L.totalB = b;
  return L;
}

struct SearchRun {
  std::vector<HostScenario> hs;
  std::vector<fpk::Scenario> scs;
  std::vector<Layout> lay;
};

// Starts the row-major copy of the resident table on the context's second
// stream (after the work already queued on the main stream). Skipped when
// the memory is not there; searches then run without it or make their own.
void start_costT(fp_ctx* ctx) {
  if (!ctx->row_copy) return;
  if (const char* e = std::getenv("FLEETPLACE_COST_T"))
    if (std::atoi(e) == 0) return;
  const size_t need = (size_t)std::max(ctx->M, 0) * (size_t)std::max(ctx->B, 0);
  if (need == 0) return;
  if (ctx->costT_cap < need) {
    if (ctx->d_costT) cudaFree(ctx->d_costT);
    ctx->d_costT = nullptr;
    ctx->costT_cap = 0;
    if (cudaMalloc(&ctx->d_costT, sizeof(double) * need) != cudaSuccess) {
      cudaGetLastError();
      ctx->d_costT = nullptr;
      return;
    }
    ctx->costT_cap = need;
  }
  if (!ctx->aux) check(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking), "stream");
  if (!ctx->table_ready)
    check(cudaEventCreateWithFlags(&ctx->table_ready, cudaEventDisableTiming), "event");
  if (!ctx->costT_ready)
    check(cudaEventCreateWithFlags(&ctx->costT_ready, cudaEventDisableTiming), "event");
  if (!ctx->copy_t0) check(cudaEventCreate(&ctx->copy_t0), "event");
  if (!ctx->copy_t1) check(cudaEventCreate(&ctx->copy_t1), "event");
  check(cudaEventRecord(ctx->table_ready, ctx->stream), "event");
  check(cudaStreamWaitEvent(ctx->aux, ctx->table_ready, 0), "wait");
  check(cudaEventRecord(ctx->copy_t0, ctx->aux), "event");
  check(fpk::launch_transpose(ctx->d_cost, ctx->M, ctx->B, ctx->d_costT, ctx->aux), "transpose");
  check(cudaEventRecord(ctx->copy_t1, ctx->aux), "event");
  check(cudaEventRecord(ctx->costT_ready, ctx->aux), "event");
  ctx->copy_timed = true;
  ctx->launches += 1;
  ctx->costT_valid = true;
}

// FLEETPLACE_TRACE=1: host-side timestamps of a search on stderr.
struct Trace {
  bool on = std::getenv("FLEETPLACE_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) const {
    if (!on) return;
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[fleetplace trace] %8.3f ms  %s\n", ms, what);
  }
};

// Shared driver for fp_search / fp_search_batch. `tables[s]` is a device
// pointer to scenario s's table (nullptr = the scenario's arena copy).
// sweep != nullptr (fp_neighbourhood_sweep): stop after the search start's
// neighbourhood sweep and hand out its tables instead of searching.
void run_search(fp_ctx* ctx, int n, const fp_instance* insts, const fp_search_config* cfgs,
                const fp_search_start* starts, fp_search_result* outs,
                const std::vector<const double*>& dev_tables,
                const std::vector<const double*>& host_tables,
                fp_sweep_result* sweep = nullptr) {
  const int M = insts[0].n_missions;
  for (int s = 1; s < n; ++s)
    if (insts[s].n_missions != M)
      throw FpError(FP_ERR_INVALID_ARGUMENT, "batch scenarios must share the mission count");
  // per-scenario SearchConfig (tabu_search / local_search preconditions,
  // proj/src/search.cpp:438-460); scenarios with the same seed share one
  // permutation stream (the stream depends on the seed and M only)
  std::vector<long long> tenures(n);
  std::vector<int> pstream(n);
  std::vector<uint64_t> seeds;
  int max_passes_all = -2;  // the largest cap (-1: some scenario has none)
  bool any_tabu = false, any_debug = false;
  {
    std::unordered_map<uint64_t, int> sidx;
    for (int s = 0; s < n; ++s) {
      const fp_search_config* c = &cfgs[s];
      if (c->mode != FP_MODE_LOCAL && c->mode != FP_MODE_TABU)
        throw FpError(FP_ERR_INVALID_ARGUMENT, "unknown search mode");
      tenures[s] = resolve_tenure(c, M);
      any_tabu |= c->mode == FP_MODE_TABU;
      any_debug |= c->debug_check_deltas != 0;
      auto it = sidx.emplace(c->seed, (int)seeds.size());
      if (it.second) seeds.push_back(c->seed);
      pstream[s] = it.first->second;
      max_passes_all = c->max_passes < 0 || max_passes_all == -1 ? -1 : std::max(max_passes_all, c->max_passes);
    }
  }
  const int D = (int)seeds.size();
  cudaStream_t st = ctx->stream;
  const Trace tr;

  SearchRun run;
  run.hs.resize(n);
  parallel_for(n, [&](int s) { run.hs[s] = prepare(&insts[s], &starts[s]); });

  // ---- arena
  size_t totalA = 0, totalB = 0;
  run.lay.resize(n);
  std::vector<size_t> baseA(n), baseB(n);
  int maxV = 0, maxB = 0, maxK = 0;
  for (int s = 0; s < n; ++s) {
    const HostScenario& h = run.hs[s];
    const int V = insts[s].n_vehicles, B = insts[s].n_bases;
    maxV = std::max(maxV, V);
    maxB = std::max(maxB, B);
    maxK = std::max(maxK, h.K);
    run.lay[s] = layout(M, B, V, h.K, h.psize + V + 1, dev_tables[s] == nullptr);
    baseA[s] = totalA;
    totalA += run.lay[s].totalA;
    baseB[s] = totalB;
    totalB += run.lay[s].totalB;
  }
  tr.mark("prepared");
  // Small scenarios run many passes per launch, each block rebuilding its
  // own mirrors/bitsets between passes (scenarios of a batch progress
  // independently); large ones run one pass per launch after the grid-wide
  // sweep. Permutations for a chunk of passes are generated on the host
  // while the device runs the previous chunk.
  // (single scenarios: one block rebuilding its bitsets is slower than the
  // grid-wide sweep plus a relaunch once V*M passes 64K)
  bool inkernel = n > 1 || (long long)maxV * M <= (64ll << 10);
  if (const char* e = std::getenv("FLEETPLACE_INKERNEL")) inkernel = n > 1 || std::atoi(e) != 0;
  // passes per host round trip: in-kernel mode runs them in one launch; the
  // sweep mode enqueues (sweep, pass) launch pairs that exit at once when the
  // scenario is done, so the host only synchronises once per chunk
  // In-kernel chunks hold up to 1024 passes (64 MB of permutations); a
  // single scenario's chunks grow 32, 64, ... so a short search generates
  // few permutations.
  // (several permutation streams: their chunks share a budget of up to 16x
  // one stream's, permutations and device draws together)
  // (one stream: 1024 passes of c5's 5k missions, ~123 MB, so a batch runs in
  // one launch and no scenario waits at a chunk boundary)
  const long long budget = ((inkernel ? 192ll : 16ll) << 20) * std::min(D, 16);
  const long long per_pass = (inkernel ? 24ll : 8ll) * std::max(M, 1) * D;
  int kmax = (int)std::max<long long>(1, std::min<long long>(inkernel ? 1024 : 16, budget / per_pass));
  if (const char* e = std::getenv("FLEETPLACE_KPASSES")) kmax = std::max(1, std::atoi(e));
  const size_t chunk_ints = 2ull * kmax * M * D + 2;
  // ---- device workspace (owned by the context, reused across calls):
  // arena | row-major table copies | counters | scenarios | active | perms.
  // The row-major copy of each table (mission-major: one mission's costs at
  // every base contiguous) serves the per-move updates that run over bases;
  // it is left out when memory is short (FLEETPLACE_COST_T=0 disables it).
  bool cost_t = true;
  if (const char* e = std::getenv("FLEETPLACE_COST_T")) cost_t = std::atoi(e) != 0;
  // a single search on the context's own table keeps its copy with the
  // table (made once, reused by every later search on it)
  const bool ctx_copy = cost_t && n == 1 && ctx->d_cost && dev_tables[0] == ctx->d_cost;
  if (ctx_copy && ctx->costT_cap < (size_t)M * insts[0].n_bases) {
    if (ctx->d_costT) {
      cudaStreamSynchronize(st);
      if (ctx->aux) cudaStreamSynchronize(ctx->aux);
      cudaFree(ctx->d_costT);
    }
    ctx->d_costT = nullptr;
    ctx->costT_cap = 0;
    ctx->costT_valid = false;
    if (cudaMalloc(&ctx->d_costT, sizeof(double) * (size_t)M * insts[0].n_bases) == cudaSuccess) {
      ctx->costT_cap = (size_t)M * insts[0].n_bases;
    } else {
      cudaGetLastError();
      ctx->d_costT = nullptr;
      cost_t = false;
    }
  }
  size_t tt = 0;
  std::vector<size_t> tbase(n, 0);
  for (int s = 0; s < n; ++s) {
    tbase[s] = tt;
    tt += (size_t)M * insts[s].n_bases;
  }
  const size_t o_B = align_up(totalA), o_ctr = align_up(o_B + totalB), o_scs = align_up(o_ctr + sizeof(fpk::Counters) * n),
               o_act = align_up(o_scs + sizeof(fpk::Scenario) * n),
               o_perm = align_up(o_act + 4ull * n), o_mt = align_up(o_perm + 4ull * chunk_ints),
               o_pbad = align_up(o_mt + sizeof(fpk::MtState) * D),
               o_draws = align_up(o_pbad + sizeof(int)),
               o_costT = align_up(o_draws + (inkernel ? 16ull * kmax * (size_t)std::max(M - 1, 0) * D : 0));
  auto ws_get = [&](size_t bytes) -> bool {
    if (bytes <= ctx->ws_cap) return true;
    if (ctx->ws) {
      cudaStreamSynchronize(st);
      cudaFree(ctx->ws);
    }
    ctx->ws = nullptr;
    ctx->ws_cap = 0;
    const size_t want = bytes + bytes / 8;
    if (cudaMalloc(&ctx->ws, want) != cudaSuccess) {
      cudaGetLastError();
      ctx->ws = nullptr;
      return false;
    }
    ctx->ws_cap = want;
    return true;
  };
  if (!(cost_t && ws_get(o_costT + (ctx_copy ? 0 : 8ull * tt)))) {
    cost_t = false;
    if (!ws_get(o_costT)) throw FpError(FP_ERR_OUT_OF_MEMORY, "search workspace");
  }
  unsigned char* const d0 = ctx->ws;
  fpk::Counters* const d_ctr = reinterpret_cast<fpk::Counters*>(d0 + o_ctr);
  fpk::Scenario* const d_scs = reinterpret_cast<fpk::Scenario*>(d0 + o_scs);
  int32_t* const d_active = reinterpret_cast<int32_t*>(d0 + o_act);
  int32_t* const d_perm = reinterpret_cast<int32_t*>(d0 + o_perm);
  double* const d_costT = reinterpret_cast<double*>(d0 + o_costT);
  fpk::MtState* const d_mt = reinterpret_cast<fpk::MtState*>(d0 + o_mt);
  int* const d_pbad = reinterpret_cast<int*>(d0 + o_pbad);
  unsigned long long* const d_draws = reinterpret_cast<unsigned long long*>(d0 + o_draws);
  const size_t small_bytes = sizeof(fpk::Counters) * n + 4ull * n + 64;
  if (ctx->h_small_cap < small_bytes) {
    if (ctx->h_small) cudaFreeHost(ctx->h_small);
    ctx->h_small = nullptr;
    ctx->h_small_cap = 0;
    check(cudaMallocHost(&ctx->h_small, small_bytes), "pinned control words");
    ctx->h_small_cap = small_bytes;
  }
  fpk::Counters* const ctrs = reinterpret_cast<fpk::Counters*>(ctx->h_small);
  int32_t* const active = reinterpret_cast<int32_t*>(ctx->h_small + sizeof(fpk::Counters) * n);
  int* const pbad_h = reinterpret_cast<int*>(ctx->h_small + sizeof(fpk::Counters) * n + 4ull * n);
  for (int s = 0; s < n; ++s) {
    ctrs[s] = fpk::Counters{};
    ctrs[s].psize = run.hs[s].psize;
    // test hook: every accept decision through the exact sums (same results)
    if (const char* e = std::getenv("FLEETPLACE_FORCE_EXACT")) ctrs[s].force_exact = std::atoi(e);
    if (const char* e = std::getenv("FLEETPLACE_HELPED_CHAINS")) ctrs[s].chain_mode = std::atoi(e) == 0;
    if (const char* e = std::getenv("FLEETPLACE_CHECK_IMPT")) ctrs[s].check_impt = std::atoi(e);
  }
  // region A of every scenario, staged in the context's pinned buffer
  if (ctx->h_stage_cap < totalA) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_cap = 0;
    check(cudaMallocHost(&ctx->h_stage, totalA + totalA / 4), "pinned stage");
    ctx->h_stage_cap = totalA + totalA / 4;
  }
  unsigned char* const stage = ctx->h_stage;
  std::memset(stage, 0, totalA);
  run.scs.resize(n);
  parallel_for(n, [&](int s) {
    const HostScenario& h = run.hs[s];
    const Layout& L = run.lay[s];
    const fp_instance* in = &insts[s];
    const int V = in->n_vehicles, B = in->n_bases;
    unsigned char* hb = stage + baseA[s];
    unsigned char* db = d0 + baseA[s];              // region A (staged)
    unsigned char* dw = d0 + o_B + baseB[s];        // region B (device-built)
    if (M) std::memcpy(hb + L.ro, in->rotary_only, M);
    if (V) std::memcpy(hb + L.vfixed, h.vfixed.data(), V);
    if (B) std::memcpy(hb + L.bheli, h.bheli.data(), B);
    if (V) std::memcpy(hb + L.vrk, h.vrk.data(), 4ull * V);
    if (B) std::memcpy(hb + L.brk, h.brk.data(), 4ull * B);
    if (M) std::memcpy(hb + L.mv, h.mv.data(), 4ull * M);
    if (V) std::memcpy(hb + L.vbase, h.vbase.data(), 4ull * V);
    if (V) std::memcpy(hb + L.vcount, h.vcount.data(), 4ull * V);
    if (B) std::memcpy(hb + L.bveh, h.bveh.data(), 4ull * B);
    if (h.psize) std::memcpy(hb + L.pkind, h.pkind.data(), 4ull * h.psize);
    if (h.psize) std::memcpy(hb + L.pidx, h.pidx.data(), 4ull * h.psize);

    fpk::Scenario& S = run.scs[s];
    S.cost = dev_tables[s] ? dev_tables[s] : reinterpret_cast<const double*>(dw + L.cost);
    S.costT = !cost_t ? nullptr : ctx_copy ? ctx->d_costT : d_costT + tbase[s];
    S.ro = db + L.ro;
    S.vfixed = db + L.vfixed;
    S.bheli = db + L.bheli;
    S.vrk = reinterpret_cast<const int32_t*>(db + L.vrk);
    S.brk = reinterpret_cast<const int32_t*>(db + L.brk);
    S.mv = reinterpret_cast<int32_t*>(db + L.mv);
    S.mc = reinterpret_cast<double*>(dw + L.mc);
    S.vbase = reinterpret_cast<int32_t*>(db + L.vbase);
    S.vcount = reinterpret_cast<int32_t*>(db + L.vcount);
    S.bveh = reinterpret_cast<int32_t*>(db + L.bveh);
    S.pkind = reinterpret_cast<int32_t*>(db + L.pkind);
    S.pidx = reinterpret_cast<int32_t*>(db + L.pidx);
    S.mvp = reinterpret_cast<int32_t*>(dw + L.mvp);
    S.mcp = reinterpret_cast<double*>(dw + L.mcp);
    S.rop = dw + L.rop;
    S.invb = reinterpret_cast<int32_t*>(dw + L.invb);
    S.exp_take = reinterpret_cast<long long*>(db + L.exp_take);
    S.exp_reas = reinterpret_cast<long long*>(db + L.exp_reas);
    S.exp_rel = reinterpret_cast<long long*>(db + L.exp_rel);
    S.role_rel = db + L.role_rel;
    S.rA = reinterpret_cast<double*>(dw + L.rA);
    S.rE = reinterpret_cast<double*>(dw + L.rE);
    S.rU = reinterpret_cast<double*>(dw + L.rU);
    S.rcnt = reinterpret_cast<int32_t*>(dw + L.rcnt);
    S.imp = reinterpret_cast<uint32_t*>(dw + L.imp);
    S.mem = reinterpret_cast<uint32_t*>(dw + L.mem);
    S.scratch = reinterpret_cast<int32_t*>(dw + L.scratch);
    S.hc = reinterpret_cast<fpk::HelperCtl*>(db + L.hc);
    S.hdelta = reinterpret_cast<int32_t*>(db + L.hdelta);
    S.hsum = reinterpret_cast<double*>(db + L.hsum);
    S.habs = reinterpret_cast<double*>(db + L.habs);
    S.hec = reinterpret_cast<int32_t*>(db + L.hec);
    S.hrs = reinterpret_cast<long long*>(dw + L.hrs);
    S.hue = reinterpret_cast<int32_t*>(dw + L.hue);
    S.impT = reinterpret_cast<uint32_t*>(dw + L.impT);
    S.vseg = reinterpret_cast<int32_t*>(dw + L.vseg);
    S.vcur = reinterpret_cast<int32_t*>(dw + L.vcur);
    S.vch = reinterpret_cast<int32_t*>(dw + L.vch);
    S.hlog = reinterpret_cast<fpk::SubRec*>(dw + L.hlog);
    S.hP = reinterpret_cast<double*>(dw + L.hP);
    S.hP2 = reinterpret_cast<double*>(dw + L.hP2);
    S.nvw = (V + 31) / 32;
    {
      const size_t nsub = ((size_t)M + fpk::kChainSub - 1) / fpk::kChainSub + 1;
      int32_t* he = reinterpret_cast<int32_t*>(hb + L.hec);
      for (size_t c = 0; c < nsub; ++c) he[c] = fpk::kNoBinade;
    }
    S.nwd = (M + 31) / 32;
    S.ctr = d_ctr + s;
    S.M = M;
    S.B = B;
    S.V = V;
    S.K = h.K;
    S.pool_cap = h.psize + V + 1;
    S.tenure = tenures[s];
    S.max_passes = cfgs[s].max_passes < 0 ? -1 : cfgs[s].max_passes;
    S.tabu = cfgs[s].mode == FP_MODE_TABU;
    S.debug = cfgs[s].debug_check_deltas != 0;
    S.pstream = pstream[s];
  });
  cudaEvent_t ev0, ev1;
  check(cudaEventCreate(&ev0), "event");
  check(cudaEventCreate(&ev1), "event");
  // host tables (batches): straight from the caller's buffers into the
  // device region, before the timed search
  {
    // caller tables: uploaded, then checked on the device (distances: finite, >= 0)
    std::vector<const double*> cp;
    std::vector<long long> cn;
    long long mx = 0;
    for (int s = 0; s < n; ++s)
      if (!dev_tables[s] && (size_t)M * insts[s].n_bases) {
        h2d(const_cast<double*>(run.scs[s].cost), host_tables[s], (size_t)M * insts[s].n_bases, st);
        cp.push_back(run.scs[s].cost);
        cn.push_back((long long)M * insts[s].n_bases);
        mx = std::max(mx, cn.back());
      }
    if (!cp.empty()) {
      const int k = (int)cp.size();
      DBuf<unsigned char> tmp(16ull * k + 4ull * k, st);
      const double** d_p = reinterpret_cast<const double**>(tmp.p);
      long long* d_n = reinterpret_cast<long long*>(tmp.p + 8ull * k);
      int* d_bad = reinterpret_cast<int*>(tmp.p + 16ull * k);
      h2d(d_p, cp.data(), k, st);
      h2d(d_n, cn.data(), k, st);
      check(fpk::launch_table_check_multi(d_p, d_n, k, mx, d_bad, st), "table_check");
      std::vector<int> bad(k);
      d2h(bad.data(), d_bad, k, st);
      check(cudaStreamSynchronize(st), "table check sync");
      for (int x : bad)
        if (x)
          throw FpError(FP_ERR_INVALID_ARGUMENT,
                        "the search needs distance tables whose entries are finite and >= 0");
      ctx->launches += 1;
    }
  }
  check(cudaEventRecord(ev0, st), "event");
  h2d(d0, stage, totalA, st);
  h2d(d_scs, run.scs.data(), n, st);
  for (int s = 0; s < n; ++s) active[s] = 1;
  h2d(d_ctr, ctrs, n, st);
  // pinned staging of host-generated permutations (device-drawn ones need none)
  auto host_perm_buffers = [&]() {
    if (ctx->perm_cap >= chunk_ints) return;
    for (auto& p : ctx->h_perm)
      if (p) cudaFreeHost(p), p = nullptr;
    for (auto& p : ctx->h_perm) check(cudaMallocHost(&p, sizeof(int32_t) * chunk_ints), "pinned");
    ctx->perm_cap = chunk_ints;
  };
  double init_ms = 0.0, sweep_ms = 0.0, pass_ms = 0.0;
  uint64_t pass_launches = 0;
  cudaEvent_t ei[5];
  for (auto& e : ei) check(cudaEventCreate(&e), "event");
  const bool transpose = cost_t && !(ctx_copy && ctx->costT_valid);
  // a copy made on the second stream is waited for; one an earlier search
  // made in-stream (no eager copy, or its allocation failed) is ordered already
  if (cost_t && ctx_copy && ctx->costT_valid && ctx->costT_ready)
    check(cudaStreamWaitEvent(st, ctx->costT_ready, 0), "wait");
  // (a sweep alone does not need the exact start total)
  if (std::getenv("FLEETPLACE_INIT_SIDE") && !ctx->aux)
    check(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking), "stream");
  check(fpk::launch_init(d_scs, run.scs.data(), n, M, maxB, maxV, transpose, st, ei, !sweep,
                         ctx->aux),
        "init_kernel");
  if (ctx_copy && cost_t) ctx->costT_valid = true;
  const bool rows_stream = n == 1 && cost_t && M > 0 && maxB > 0 && maxV > 0;
  ctx->launches += 1 + (M > 0 ? 2 : 0) + (rows_stream ? 4 : (maxB > 0 ? 1 : 0)) +
                   (transpose && M > 0 && maxB > 0 ? 1 : 0);
  tr.mark("allocated, staged, init launched");
  if (sweep) {
    // the sweep's results of scenario 0, then done
    const fpk::Scenario& S = run.scs[0];
    const int V = insts[0].n_vehicles, B = insts[0].n_bases;
    const size_t bv = (size_t)B * V, nw = (size_t)M * S.nvw;
    const cudaMemcpyKind k = sweep->device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    auto out = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) check(cudaMemcpyAsync(dst, src, bytes, k, st), "sweep copy");
    };
    out(sweep->reloc_sum, S.rA, 8 * bv);
    out(sweep->reloc_err, S.rE, 8 * bv);
    out(sweep->reloc_abs, S.rU, 8 * bv);
    out(sweep->improve_rows, S.impT, 4 * nw);
    out(sweep->mission_cost, S.mc, 8ull * M);
    check(cudaStreamSynchronize(st), "sweep sync");
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ei[2], ei[4]);
    cudaEventElapsedTime(&b, ei[0], ei[4]);
    sweep->sweep_ms = a;
    sweep->total_ms = b;
    for (auto& e : ei) cudaEventDestroy(e);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return;
  }
  std::vector<cudaEvent_t> sweep_ev;  // (start, end) pairs around grid-wide sweeps
  std::vector<cudaEvent_t> pass_ev;   // (start, end) pairs around pass-kernel launches
  std::vector<PermStream> rngs;
  for (uint64_t sd : seeds) rngs.emplace_back(sd);
  // a chunk of kk passes: stream d's 2*kk permutations at d * 2*kk*M
  std::vector<uint64_t> raw_draws;
  auto gen_chunk = [&](int32_t* buf, int kk) {
    for (int d = 0; d < D; ++d) rngs[d].perms(M, 2 * kk, buf + 2ll * kk * d * M, raw_draws);
  };
  long long launched = 0;  // passes whose permutations went to the device
  // batches: one launch for (nearly) every search — a chunk boundary makes
  // every scenario wait for the slowest; single scenarios start small
  int threads = n == 1 ? 512 : 256;
  if (const char* e = std::getenv("FLEETPLACE_THREADS")) threads = std::atoi(e);
  int threads_later = 0;
  if (const char* e = std::getenv("FLEETPLACE_THREADS_LATER")) threads_later = std::atoi(e);
  // medium single scenarios (8k <= M < 32k, bitsets in shared memory): the
  // relocation-heavy first passes run with helper blocks (bitsets in global
  // memory, the relocations' O(M) work spread over the SMs), one pass per
  // launch, until a pass applies fewer than two relocations; the rest run in
  // one block with the bitsets in shared memory. An execution strategy only:
  // results are identical either way (c2: first 3 passes 5.25 -> ~4.9 ms).
  bool adaptive = n == 1 && !inkernel && M >= (8 << 10) && M < (32 << 10) && threads < 1024 &&
                  !std::getenv("FLEETPLACE_HELPERS");
  if (const char* e = std::getenv("FLEETPLACE_ADAPTIVE_HELPERS")) adaptive = adaptive && std::atoi(e) != 0;
  // (large single scenarios start with 2 passes: the GPU starts after the first
  // chunk of host permutations, later chunks are drawn while it works)
  int kfirst = inkernel ? (n == 1 ? std::min(kmax, 32) : kmax) : (adaptive ? 1 : std::min(kmax, 2));
  if (const char* e = std::getenv("FLEETPLACE_KFIRST")) kfirst = std::max(1, std::min(kmax, std::atoi(e)));
  auto next_chunk = [&](int prev) {
    int k = prev == 0 ? kfirst : (adaptive ? 1 : std::min(kmax, 2 * prev));
    if (max_passes_all >= 0) k = (int)std::max<long long>(1, std::min<long long>(k, max_passes_all - launched));
    return k;
  };
  // In-kernel mode draws the permutations on the device (perm_kernels.cu):
  // the host stream is the bottleneck of batches. The host generator stays
  // the fallback (a rejected draw, FLEETPLACE_DEVICE_PERMS=0).
  bool dev_perm = inkernel && M >= 2 && fpk::fy_smem_bytes(M) <= (200u << 10);
  if (const char* e = std::getenv("FLEETPLACE_DEVICE_PERMS")) dev_perm = dev_perm && std::atoi(e) != 0;
  bool force_bad = std::getenv("FLEETPLACE_PERM_FORCE_BAD") != nullptr;  // test hook
  // the first chunk's draws depend on the seeds only: on a side stream they
  // overlap the staging and init kernels (c5 share: ~10 ms of draws)
  cudaStream_t pst = st;
  cudaEvent_t perm_done = nullptr;
  if (dev_perm && inkernel) {
    if (!ctx->pstream) {
      // highest priority: the draws' single block is dispatched ahead of the
      // start kernels' blocks queued on the search stream
      int least = 0, greatest = 0;
      check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
      check(cudaStreamCreateWithPriority(&ctx->pstream, cudaStreamNonBlocking, greatest), "stream");
    }
    pst = ctx->pstream;
    check(cudaEventCreateWithFlags(&perm_done, cudaEventDisableTiming), "event");
  }
  if (dev_perm) {
    // seeded on the device: no host copy queued in front of the draws
    check(fpk::launch_mt_seed(d_mt, reinterpret_cast<const unsigned long long*>(seeds.data()), D, pst),
          "mt_seed");
    check(cudaMemsetAsync(d_pbad, 0, sizeof(int), pst), "memset");
  }
  int kchunk = next_chunk(0);
  int buf = 0;
  if (!dev_perm) {
    host_perm_buffers();
    gen_chunk(ctx->h_perm[buf], kchunk);  // overlaps the init kernels
  }
  tr.mark("first permutation chunk");
  // large single scenarios share each relocation's O(M) work with helper
  // blocks (-1 = as many as fit; FLEETPLACE_HELPERS=0 disables)
  int helpers = n == 1 && M >= (32 << 10) ? -1 : 0;
  if (const char* e = std::getenv("FLEETPLACE_HELPERS")) helpers = std::atoi(e);
  // the 1024-thread variant (a FLEETPLACE_THREADS experiment knob, 64
  // registers, ~1 KB of spills) never runs with helper blocks: that pairing
  // faults (illegal instruction) in some builds and not in others
  if (threads >= 1024) helpers = 0;
  unsigned epoch = 0;
  int n_active = n;
  bool active_dirty = true;  // the device copy of `active` is stale
  while (n_active > 0) {
    if (active_dirty) h2d(d_active, active, n, st);
    active_dirty = false;
    if (dev_perm) {
      cudaEvent_t q0 = nullptr, q1 = nullptr;
      if (tr.on) {
        cudaEventCreate(&q0);
        cudaEventCreate(&q1);
        cudaEventRecord(q0, pst);
      }
      check(fpk::launch_permutations(d_mt, D, M, 2 * kchunk, d_draws, d_perm, d_pbad, pst),
            "permutations");
      if (pst != st) {
        check(cudaEventRecord(perm_done, pst), "event");
        check(cudaStreamWaitEvent(st, perm_done, 0), "wait");
        pst = st;  // later chunks: in order on the search stream
      }
      if (tr.on) {
        cudaEventRecord(q1, st);
        cudaEventSynchronize(q1);
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev0, q0);
        cudaEventElapsedTime(&b, q0, q1);
        std::fprintf(stderr, "[fleetplace trace] device: start->perms %.3f ms, perms %.3f ms (%d passes)\n", a, b, kchunk);
        cudaEventDestroy(q0);
        cudaEventDestroy(q1);
      }
      ctx->launches += 2;
      if (force_bad) check(cudaMemsetAsync(d_pbad, 1, 1, st), "memset");
    } else {
      h2d(d_perm, ctx->h_perm[buf], 2ull * kchunk * M * D, st);
    }
    if (inkernel) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      check(fpk::launch_pass(d_scs, d_active, n, d_perm, kchunk, true,
                             max_passes_all, M, any_tabu, tenures[0], any_debug, maxV,
                             maxB, maxK, st, threads, 0, 0u, dev_perm ? d_pbad : nullptr),
            "pass_kernel");
      cudaEventRecord(e1, st);
      pass_ev.push_back(e0);
      pass_ev.push_back(e1);
      ctx->launches += 1;
      pass_launches += 1;
    } else {
      for (int k = 0; k < kchunk; ++k) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        check(fpk::launch_sweep(d_scs, d_active, n, d_perm + 2ll * k * M, M, st),
              "prep_kernel");
        cudaEventRecord(e1, st);
        sweep_ev.push_back(e0);
        sweep_ev.push_back(e1);
        check(fpk::launch_pass(d_scs, d_active, n, d_perm + 2ll * k * M, 1,
                               false, max_passes_all, M, any_tabu, tenures[0],
                               any_debug, maxV, maxB, maxK, st, threads,
                               adaptive ? -1 : helpers, ++epoch, nullptr, adaptive),
              "pass_kernel");
        cudaEvent_t e2;
        cudaEventCreate(&e2);
        cudaEventRecord(e2, st);
        pass_ev.push_back(e1);
        pass_ev.push_back(e2);
        ctx->launches += M > 0 ? 2 : 1;
        pass_launches += 1;
      }
    }
    // next chunk's permutations while the device works
    launched += kchunk;
    const int knext = next_chunk(kchunk);
    const int nb = buf ^ 1;
    if (!dev_perm) gen_chunk(ctx->h_perm[nb], knext);
    d2h(ctrs, d_ctr, n, st);
    *pbad_h = 0;
    if (dev_perm) d2h(pbad_h, d_pbad, 1, st);
    wait_stream(st, inkernel, "pass sync");
    for (size_t e = 0; e + 1 < pass_ev.size(); e += 2) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pass_ev[e], pass_ev[e + 1]);
      pass_ms += ms;
      // (in sweep mode the start event is the sweep's end event, destroyed below)
      if (inkernel) cudaEventDestroy(pass_ev[e]);
      cudaEventDestroy(pass_ev[e + 1]);
    }
    pass_ev.clear();
    for (size_t e = 0; e + 1 < sweep_ev.size(); e += 2) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, sweep_ev[e], sweep_ev[e + 1]);
      sweep_ms += ms;
      cudaEventDestroy(sweep_ev[e]);
      cudaEventDestroy(sweep_ev[e + 1]);
    }
    sweep_ev.clear();
    if (*pbad_h) {
      // a rejected draw (or the test hook): the pass kernel did not run this
      // chunk; regenerate the stream exactly on the host and redo the chunk
      dev_perm = false;
      force_bad = false;
      launched -= kchunk;
      std::vector<int32_t> skip((size_t)std::max(M, 1));
      for (int d = 0; d < D; ++d) {
        rngs[d] = PermStream(seeds[d]);
        for (long long p = 0; p < 2 * launched; ++p) rngs[d].perm(M, skip.data());
      }
      host_perm_buffers();
      gen_chunk(ctx->h_perm[buf], kchunk);
      tr.mark("device permutation chunk rejected: host stream");
      continue;
    }
    buf = nb;
    kchunk = knext;
    if (threads_later > 0) threads = threads_later;
    if (adaptive && ctrs[0].pass_relocs < 2) adaptive = false;
    tr.mark("chunk synchronised");
    for (int s = 0; s < n; ++s) {
      if (!active[s]) continue;
      if (ctrs[s].done || ctrs[s].error) {
        active[s] = 0;
        --n_active;
        active_dirty = true;
      }
    }
  }
  if (perm_done) cudaEventDestroy(perm_done);  // (the wait on it is enqueued)
  check(fpk::launch_final(d_scs, n, st), "final_kernel");
  ctx->launches += 1;
  check(cudaEventRecord(ev1, st), "event");
  d2h(ctrs, d_ctr, n, st);
  if (n < 64) {
    for (int s = 0; s < n; ++s) {
      d2h(outs[s].vehicle_base, run.scs[s].vbase, insts[s].n_vehicles, st);
      d2h(outs[s].mission_vehicle, run.scs[s].mv, (size_t)M, st);
    }
    wait_stream(st, inkernel, "final sync");
  } else {
    // large batches: every scenario's result gathered on the device, one copy
    // into the pinned stage (region A, already consumed), spread on threads
    std::vector<long long> vbo(n + 1, 0);
    for (int s = 0; s < n; ++s) vbo[s + 1] = vbo[s] + insts[s].n_vehicles;
    const size_t nres = (size_t)n * M + (size_t)vbo[n];
    DBuf<unsigned char> dres(4 * nres + 8ull * (n + 1), st);
    int32_t* d_mv = reinterpret_cast<int32_t*>(dres.p);
    int32_t* d_vb = d_mv + (size_t)n * M;
    long long* d_vbo = reinterpret_cast<long long*>(dres.p + 4 * nres);
    h2d(d_vbo, vbo.data(), n + 1, st);
    check(fpk::launch_gather_results(d_scs, n, M, d_mv, d_vb, d_vbo, st), "gather_results");
    ctx->launches += 1;
    int32_t* h_res = reinterpret_cast<int32_t*>(stage);  // totalA >= 4 * nres
    d2h(h_res, d_mv, nres, st);
    wait_stream(st, inkernel, "final sync");
    parallel_for(n, [&](int s) {
      std::memcpy(outs[s].mission_vehicle, h_res + (size_t)s * M, 4ull * M);
      std::memcpy(outs[s].vehicle_base, h_res + (size_t)n * M + vbo[s], 4ull * insts[s].n_vehicles);
    });
  }
  tr.mark("final sync");
  double init_part[4] = {0, 0, 0, 0};
  {
    float ims = 0.f;
    cudaEventElapsedTime(&ims, ei[0], ei[4]);
    init_ms = ims;
    for (int k = 0; k < 4; ++k) {
      cudaEventElapsedTime(&ims, ei[k], ei[k + 1]);
      init_part[k] = ims;
    }
    for (auto& e : ei) cudaEventDestroy(e);
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  for (int s = 0; s < n; ++s) {
    const fpk::Counters& c = ctrs[s];
    if (c.error == FP_ERR_INFEASIBLE)
      throw FpError(FP_ERR_INFEASIBLE, "infeasible assignment during debug_check_deltas");
    if (c.error == FP_ERR_LOGIC)
      throw FpError(FP_ERR_LOGIC, "incremental objective drifted from recomputation");
    if (c.error) throw FpError((fp_status)c.error, "search failed");
    fp_search_stats& o = outs[s].stats;
    o.passes = (uint64_t)c.passes;
    o.evaluations = c.evaluations;
    o.applied_moves = c.applied;
    o.committed_moves = c.applied;
    o.tabu_skips_outer = c.skips_outer;
    o.tabu_skips_inner = c.skips_inner;
    o.final_objective_km = c.final_total;
    outs[s].device_ms = ms;
    outs[s].exact_fallbacks = c.fallbacks;
    outs[s].init_ms = init_ms;
    for (int k = 0; k < 4; ++k) outs[s].init_part_ms[k] = init_part[k];
    outs[s].sweep_ms = sweep_ms;
    outs[s].pass_ms = pass_ms;
    outs[s].pass_launches = pass_launches;
    for (int k = 0; k < 16; ++k) outs[s].phase_cycles[k] = c.cycles[k];
    for (int k = 0; k < 5; ++k) outs[s].event_counts[k] = c.counts[k];
    outs[s].kernel_launches = ctx->launches;
  }
  tr.mark("done");
}

}  // namespace

extern "C" {

int32_t fp_abi_version(void) { return FP_ABI_VERSION; }

const char* fp_last_error(void) { return g_err.c_str(); }

fp_status fp_ctx_create(int32_t device, fp_ctx** out) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw FpError(FP_ERR_CUDA, "no CUDA device available (fleetplace_b200 has no CPU path)");
    if (device < 0 || device >= n) throw FpError(FP_ERR_INVALID_ARGUMENT, "bad device ordinal");
    check(cudaSetDevice(device), "cudaSetDevice");
    fpk::keep_pool_mapped(device);
    auto* c = new fp_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      throw CudaError(e, "cudaStreamCreate");
    }
    *out = c;
  });
}

void fp_ctx_destroy(fp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->d_cost) cudaFree(ctx->d_cost);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->aux) cudaStreamSynchronize(ctx->aux);
  if (ctx->d_costT) cudaFree(ctx->d_costT);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->h_pts) cudaFreeHost(ctx->h_pts);
  if (ctx->h_small) cudaFreeHost(ctx->h_small);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->pstream) cudaStreamDestroy(ctx->pstream);
  if (ctx->table_ready) cudaEventDestroy(ctx->table_ready);
  if (ctx->costT_ready) cudaEventDestroy(ctx->costT_ready);
  if (ctx->copy_t0) cudaEventDestroy(ctx->copy_t0);
  if (ctx->copy_t1) cudaEventDestroy(ctx->copy_t1);
  for (auto& p : ctx->h_perm)
    if (p) cudaFreeHost(p);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

uint64_t fp_ctx_kernel_launches(const fp_ctx* ctx) { return ctx ? ctx->launches : 0; }

double fp_ctx_last_kernel_ms(const fp_ctx* ctx) { return ctx ? ctx->last_kernel_ms : 0.0; }

fp_status fp_permutations(fp_ctx* ctx, uint64_t seed, int32_t n, int32_t passes, int32_t* out) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (n < 2 || passes < 0) throw FpError(FP_ERR_INVALID_ARGUMENT, "need n >= 2, passes >= 0");
    if (fpk::fy_smem_bytes(n) > (200u << 10)) throw FpError(FP_ERR_INVALID_ARGUMENT, "n too large");
    const int np = 2 * passes;
    if (np == 0) return;
    cudaStream_t st = ctx->stream;
    DBuf<fpk::MtState> d_mt(1);
    DBuf<int> d_bad(1);
    DBuf<unsigned long long> d_draws((size_t)np * (n - 1));
    DBuf<int32_t> d_perms((size_t)np * n);
    fpk::MtState seeded;
    fpk::mt_seed_host(&seeded, seed);
    h2d(d_mt.p, &seeded, 1, st);
    check(cudaMemsetAsync(d_bad.p, 0, sizeof(int), st), "memset");
    check(fpk::launch_permutations(d_mt.p, 1, n, np, d_draws.p, d_perms.p, d_bad.p, st), "perms");
    ctx->launches += 2;
    int bad = 0;
    d2h(&bad, d_bad.p, 1, st);
    d2h(out, d_perms.p, (size_t)np * n, st);
    check(cudaStreamSynchronize(st), "perm sync");
    if (bad) {  // a rejected draw: the exact host stream
      PermStream rng(seed);
      for (int p = 0; p < np; ++p) rng.perm(n, out + (size_t)p * n);
    }
  });
}

fp_status fp_ctx_set_row_copy(fp_ctx* ctx, int32_t enabled) {
  return guarded([&] {
    if (!ctx) throw FpError(FP_ERR_INVALID_ARGUMENT, "ctx is NULL");
    ctx->row_copy = enabled != 0;
  });
}

double fp_ctx_last_copy_ms(fp_ctx* ctx) {
  if (!ctx || !ctx->copy_timed) return 0.0;
  cudaSetDevice(ctx->device);
  if (cudaEventSynchronize(ctx->copy_t1) != cudaSuccess) return 0.0;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->copy_t0, ctx->copy_t1);
  return ms;
}

fp_status fp_validate_instance(const fp_instance* inst) {
  return guarded([&] { validate(inst); });
}

fp_status fp_generate_instance(uint64_t pool_seed, const double* bbox, int32_t aerodromes,
                               int32_t helipads, int32_t health_sites, int32_t missions,
                               double rotary_only_fraction, uint64_t seed, int32_t rotary,
                               int32_t fixed_wing, int32_t* base_id, uint8_t* base_kind,
                               double* base_lat, double* base_lon, int32_t* vehicle_id,
                               uint8_t* vehicle_kind, int32_t* mission_id, double* pickup_lat,
                               double* pickup_lon, double* delivery_lat, double* delivery_lon,
                               uint8_t* rotary_only) {
  return guarded([&] {
    fpk_host::generate_instance(pool_seed, bbox, aerodromes, helipads, health_sites, missions,
                                rotary_only_fraction, seed, rotary, fixed_wing, base_id,
                                base_kind, base_lat, base_lon, vehicle_id, vehicle_kind,
                                mission_id, pickup_lat, pickup_lon, delivery_lat, delivery_lon,
                                rotary_only);
    fp_instance in{aerodromes + helipads, base_id, base_kind, base_lat, base_lon,
                   rotary + fixed_wing, vehicle_id, vehicle_kind, missions, mission_id,
                   pickup_lat, pickup_lon, delivery_lat, delivery_lon, rotary_only};
    validate(&in);
  });
}

fp_status fp_build_distance_table(fp_ctx* ctx, const fp_instance* in, double radius_km,
                                  double* out_cost) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int M = in->n_missions, B = in->n_bases;
    cudaStream_t st = ctx->stream;
    if (!(radius_km >= 0.0 && radius_km < INFINITY))
      throw FpError(FP_ERR_INVALID_ARGUMENT, "radius_km must be finite and >= 0");
    Trace tr;
    table_alloc(ctx, M, B);
    tr.mark("build: table allocated");
    build_table_into(ctx, in, radius_km, ctx->d_cost);
    tr.mark("build: kernels enqueued");
    ctx->table_ok = true;  // haversine sums: finite and >= 0 for valid coordinates
    start_costT(ctx);
    if (out_cost) d2h(out_cost, ctx->d_cost, (size_t)M * B, st);
    check(cudaStreamSynchronize(st), "table sync");
    tr.mark("build: done");
  });
}

fp_status fp_haversine_batch(fp_ctx* ctx, int32_t n, const double* a_lat, const double* a_lon,
                             const double* b_lat, const double* b_lon, const double* c_lat,
                             const double* c_lon, double radius_km, double* out) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (n <= 0) return;
    const bool three = c_lat && c_lon;
    DBuf<double> d((three ? 7ull : 5ull) * n);
    double* p = d.p;
    h2d(p, a_lat, n, ctx->stream);
    h2d(p + n, a_lon, n, ctx->stream);
    h2d(p + 2ll * n, b_lat, n, ctx->stream);
    h2d(p + 3ll * n, b_lon, n, ctx->stream);
    if (three) {
      h2d(p + 5ll * n, c_lat, n, ctx->stream);
      h2d(p + 6ll * n, c_lon, n, ctx->stream);
    }
    check(fpk::launch_haversine_pairs(n, p, p + n, p + 2ll * n, p + 3ll * n,
                                      three ? p + 5ll * n : nullptr,
                                      three ? p + 6ll * n : nullptr, radius_km, p + 4ll * n,
                                      ctx->stream),
          "haversine");
    ctx->launches += 1;
    d2h(out, p + 4ll * n, n, ctx->stream);
    check(cudaStreamSynchronize(ctx->stream), "haversine sync");
  });
}

fp_status fp_table_upload(fp_ctx* ctx, int32_t n_missions, int32_t n_bases,
                          const double* cost_colmajor) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (n_missions < 0 || n_bases < 0 || ((size_t)n_missions * n_bases > 0 && !cost_colmajor))
      throw FpError(FP_ERR_INVALID_ARGUMENT, "bad table shape or NULL table");
    const Trace tr;
    table_alloc(ctx, n_missions, n_bases);
    tr.mark("upload: table allocated");
    h2d(ctx->d_cost, cost_colmajor, (size_t)n_missions * n_bases, ctx->stream);
    // a caller's matrix may hold anything: column_totals stays exact for any
    // entries, the search requires distances (checked on the device)
    ctx->table_ok = table_entries_ok(ctx, ctx->d_cost, (size_t)n_missions * n_bases, ctx->stream);
    tr.mark("upload: copied and checked");
    start_costT(ctx);
    check(cudaStreamSynchronize(ctx->stream), "upload sync");
    tr.mark("upload: done");
  });
}

fp_status fp_table_download(fp_ctx* ctx, double* out_cost) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->M < 0) throw FpError(FP_ERR_INVALID_ARGUMENT, "no resident table");
    d2h(out_cost, ctx->d_cost, (size_t)ctx->M * ctx->B, ctx->stream);
    check(cudaStreamSynchronize(ctx->stream), "download sync");
  });
}

fp_status fp_column_totals(fp_ctx* ctx, double* out_totals) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->M < 0) throw FpError(FP_ERR_INVALID_ARGUMENT, "no resident table");
    DBuf<double> d(ctx->B, ctx->stream);
    EvTimer tk(ctx->stream);
    check(fpk::launch_column_totals(ctx->d_cost, ctx->M, ctx->B, d.p, ctx->stream), "totals");
    ctx->last_kernel_ms = tk.stop_ms();
    ctx->launches += 1;
    d2h(out_totals, d.p, ctx->B, ctx->stream);
    check(cudaStreamSynchronize(ctx->stream), "totals sync");
  });
}

namespace {
// rank_bases steps (2)-(6) (rank.cpp:35-121) from the base totals `tot` on
// the resident table (the whole instance, or one mission shard of it).
void rank_from_totals(fp_ctx* ctx, const fp_instance* in, const double* tot, fp_ranked_start* out);
}  // namespace

fp_status fp_rank_bases(fp_ctx* ctx, const fp_instance* in, fp_ranked_start* out) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    validate(in);
    const int M = in->n_missions, B = in->n_bases;
    ensure_table(ctx, M, B);
    cudaStream_t st = ctx->stream;
    // (1) fixed-order column totals on the device
    DBuf<double> d_tot(B, st);
    EvTimer tk(st);
    check(fpk::launch_column_totals(ctx->d_cost, M, B, d_tot.p, st), "totals");
    ctx->last_kernel_ms = tk.stop_ms();
    ctx->launches += 1;
    d2h(out->base_totals, d_tot.p, B, st);
    check(cudaStreamSynchronize(st), "totals sync");
    rank_from_totals(ctx, in, out->base_totals, out);
  });
}

fp_status fp_column_totals_chain(fp_ctx* ctx, int32_t b0, int32_t nb, const double* carry,
                                 double* out, int32_t device_ptrs) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->M < 0) throw FpError(FP_ERR_INVALID_ARGUMENT, "no resident table");
    if (b0 < 0 || nb < 0 || (int64_t)b0 + nb > ctx->B || !out)
      throw FpError(FP_ERR_INVALID_ARGUMENT, "column range outside the resident table");
    if (nb == 0) return;
    cudaStream_t st = ctx->stream;
    const double* d_carry = carry;
    double* d_out = out;
    DBuf<double> tmp(device_ptrs ? 0 : 2 * (size_t)nb, ctx->stream);
    if (!device_ptrs) {
      d_out = tmp.p;
      if (carry) {
        h2d(tmp.p + nb, carry, nb, st);
        d_carry = tmp.p + nb;
      }
    }
    EvTimer tk(st);
    check(fpk::launch_column_totals_chain(ctx->d_cost + (size_t)b0 * ctx->M, ctx->M, nb, d_carry,
                                          d_out, st),
          "totals chain");
    ctx->last_kernel_ms = tk.stop_ms();
    ctx->launches += 1;
    if (!device_ptrs) d2h(out, d_out, nb, st);
    check(cudaStreamSynchronize(st), "totals chain sync");
  });
}

fp_status fp_rank_from_totals(fp_ctx* ctx, const fp_instance* in, const double* totals,
                              fp_ranked_start* out) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    validate(in);
    ensure_table(ctx, in->n_missions, in->n_bases);
    if (!totals) throw FpError(FP_ERR_INVALID_ARGUMENT, "totals is NULL");
    if (out->base_totals && out->base_totals != totals)
      std::copy(totals, totals + in->n_bases, out->base_totals);
    rank_from_totals(ctx, in, totals, out);
  });
}

namespace {
void rank_from_totals(fp_ctx* ctx, const fp_instance* in, const double* tot, fp_ranked_start* out) {
    const int M = in->n_missions, B = in->n_bases, V = in->n_vehicles;
    cudaStream_t st = ctx->stream;
    // (2) rank order: total ascending, lower id on ties (rank.cpp:35-43)
    std::vector<int> order(B);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      if (tot[a] != tot[b]) return tot[a] < tot[b];
      return in->base_id[a] < in->base_id[b];
    });
    int rotary = 0;
    for (int v = 0; v < V; ++v) rotary += in->vehicle_kind[v] == FP_ROTARY;
    // (3) top |fleet| with the helipad cap (rank.cpp:47-59)
    std::vector<int> chosen;
    int heli = 0;
    for (int bi : order) {
      if ((int)chosen.size() == V) break;
      const bool h = in->base_kind[bi] == FP_HELIPAD;
      if (h && heli == rotary) continue;
      chosen.push_back(bi);
      if (h) ++heli;
    }
    if ((int)chosen.size() < V)
      throw FpError(FP_ERR_VALIDATION,
                    "validation failed for bases: not enough compatible bases to place the fleet");
    // (4) placement: helipads first with rotary ids ascending (rank.cpp:61-90)
    std::vector<int> rot, fix;
    for (int v = 0; v < V; ++v) (in->vehicle_kind[v] == FP_ROTARY ? rot : fix).push_back(v);
    auto by_id = [&](int a, int b) { return in->vehicle_id[a] < in->vehicle_id[b]; };
    std::sort(rot.begin(), rot.end(), by_id);
    std::sort(fix.begin(), fix.end(), by_id);
    std::vector<int> base_vehicle(B, -1);
    for (int v = 0; v < V; ++v) out->vehicle_base[v] = -1;
    size_t nr = 0, nf = 0;
    for (int bi : chosen)
      if (in->base_kind[bi] == FP_HELIPAD) {
        const int v = rot[nr++];
        base_vehicle[bi] = v;
        out->vehicle_base[v] = bi;
      }
    for (int bi : chosen)
      if (in->base_kind[bi] != FP_HELIPAD) {
        const int v = nr < rot.size() ? rot[nr++] : fix[nf++];
        base_vehicle[bi] = v;
        out->vehicle_base[v] = bi;
      }
    // (5) per-mission argmin over occupied compatible bases (device)
    const int n = (int)chosen.size();
    std::vector<int32_t> cb(n), cbid(n), cv(n);
    std::vector<uint8_t> cf(n);
    for (int k = 0; k < n; ++k) {
      cb[k] = chosen[k];
      cbid[k] = in->base_id[chosen[k]];
      cv[k] = base_vehicle[chosen[k]];
      cf[k] = in->vehicle_kind[cv[k]] == FP_FIXED;
    }
    DBuf<int32_t> d_i32(3ull * n + (size_t)M + 1, st);
    DBuf<uint8_t> d_u8((size_t)n + M + 1, st);
    int32_t* d_cb = d_i32.p;
    int32_t* d_cbid = d_cb + n;
    int32_t* d_cv = d_cbid + n;
    int32_t* d_mv = d_cv + n;
    int32_t* d_bad = d_mv + M;
    uint8_t* d_cf = d_u8.p;
    uint8_t* d_ro = d_cf + n;
    h2d(d_cb, cb.data(), n, st);
    h2d(d_cbid, cbid.data(), n, st);
    h2d(d_cv, cv.data(), n, st);
    h2d(d_cf, cf.data(), n, st);
    // large instances: the per-mission copies through the pinned buffer
    const bool staged = (size_t)M >= (1u << 16);
    if (staged) {
      pinned_points(ctx, (size_t)M / 2 + 2);
      std::memcpy(ctx->h_pts, in->rotary_only, (size_t)M);
      h2d(d_ro, reinterpret_cast<const uint8_t*>(ctx->h_pts), M, st);
    } else {
      h2d(d_ro, in->rotary_only, M, st);
    }
    const int32_t big = 0x7fffffff;
    h2d(d_bad, &big, 1, st);
    check(fpk::launch_mission_argmin(ctx->d_cost, M, d_cb, d_cbid, d_cf, d_cv, n, d_ro, d_mv, d_bad,
                                     st),
          "mission_argmin");
    ctx->launches += 1;
    int32_t bad = 0;
    int32_t* const hmv = staged ? reinterpret_cast<int32_t*>(ctx->h_pts) : out->mission_vehicle;
    d2h(hmv, d_mv, M, st);
    d2h(&bad, d_bad, 1, st);
    check(cudaStreamSynchronize(st), "rank sync");
    if (staged)
      parallel_for(64, [&](int t) {
        const size_t lo = (size_t)M * t / 64, hi = (size_t)M * (t + 1) / 64;
        std::memcpy(out->mission_vehicle + lo, hmv + lo, 4 * (hi - lo));
      });
    if (bad != big)
      throw FpError(FP_ERR_NO_COMPATIBLE, "mission " + std::to_string(in->mission_id[bad]) +
                                              " has no compatible placed vehicle");
    // (6) unused bases in rank order (rank.cpp:118-121)
    int nu = 0;
    for (int bi : order)
      if (base_vehicle[bi] < 0) out->unused_bases[nu++] = bi;
    out->n_unused = nu;
}
}  // namespace

fp_status fp_initial_pool(const fp_instance* in, const int32_t* vehicle_base,
                          const int32_t* mission_vehicle, const int32_t* unused_bases,
                          int32_t n_unused, int32_t* out_kind, int32_t* out_index,
                          int32_t* out_size) {
  return guarded([&] {
    int k = 0;
    for (int u = 0; u < n_unused; ++u) {
      out_kind[k] = FP_POOL_EMPTY_BASE;
      out_index[k++] = unused_bases[u];
    }
    std::vector<int> served(in->n_vehicles, 0);
    for (int m = 0; m < in->n_missions; ++m)
      if (mission_vehicle[m] >= 0 && mission_vehicle[m] < in->n_vehicles) served[mission_vehicle[m]]++;
    std::vector<int> placed;
    for (int v = 0; v < in->n_vehicles; ++v)
      if (vehicle_base[v] >= 0) placed.push_back(v);
    std::sort(placed.begin(), placed.end(),
              [&](int a, int b) { return in->vehicle_id[a] < in->vehicle_id[b]; });
    for (int v : placed)
      if (!served[v]) {
        out_kind[k] = FP_POOL_IDLE_VEHICLE;
        out_index[k++] = v;
      }
    *out_size = k;
  });
}

fp_status fp_search(fp_ctx* ctx, const fp_instance* inst, const fp_search_config* cfg,
                    const fp_search_start* start, fp_search_result* out) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    ensure_table(ctx, inst->n_missions, inst->n_bases);
    if (!ctx->table_ok)
      throw FpError(FP_ERR_INVALID_ARGUMENT,
                    "the search needs a distance table whose entries are finite and >= 0");
    run_search(ctx, 1, inst, cfg, start, out, {ctx->d_cost}, {nullptr});
  });
}

fp_status fp_search_batch_configs(fp_ctx* ctx, int32_t n, const fp_instance* insts,
                                  const double* const* tables, double radius_km,
                                  const fp_search_config* cfgs, const fp_search_start* starts,
                                  fp_search_result* outs) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (n <= 0) return;
    if (!insts || !cfgs || !starts || !outs) throw FpError(FP_ERR_INVALID_ARGUMENT, "NULL batch array");
    const int M = insts[0].n_missions;
    for (int s = 1; s < n; ++s)
      if (insts[s].n_missions != M)
        throw FpError(FP_ERR_INVALID_ARGUMENT, "batch scenarios must share the mission count");
    std::vector<const double*> dev(n, nullptr), host(n, nullptr);
    // scenarios without a host table: kernel (1) for all of them in one
    // launch, into a scratch buffer (the context's resident table is untouched)
    std::vector<int> build;
    for (int s = 0; s < n; ++s) {
      if (tables && tables[s]) host[s] = tables[s];
      else build.push_back(s);
    }
    DBuf<double> built, pts;
    DBuf<fpk::TableJob> d_jobs;
    if (!build.empty()) {
      if (!(radius_km >= 0.0 && radius_km < INFINITY))
        throw FpError(FP_ERR_INVALID_ARGUMENT, "radius_km must be finite and >= 0");
      cudaStream_t st = ctx->stream;
      size_t tot = 0, npts = 0;
      int maxB = 0;
      for (int s : build) {
        tot += (size_t)M * insts[s].n_bases;
        npts += (size_t)insts[s].n_bases + 2ull * M;
        maxB = std::max(maxB, insts[s].n_bases);
      }
      built = DBuf<double>(tot + 2, st);
      // points: [lat | lon | cos] regions, each [bases, pickups, deliveries]
      // per scenario, packed on host threads into the context's pinned buffer
      pinned_points(ctx, 2 * npts);
      double* const hp = ctx->h_pts;
      pts = DBuf<double>(3 * npts + 1, st);
      std::vector<fpk::TableJob> jobs(build.size());
      std::vector<size_t> pof(build.size()), tof(build.size());
      size_t po = 0, to = 0;
      for (size_t k = 0; k < build.size(); ++k) {
        pof[k] = po;
        tof[k] = to;
        po += (size_t)insts[build[k]].n_bases + 2ull * M;
        to += (size_t)M * insts[build[k]].n_bases;
      }
      parallel_for((int)build.size(), [&](int k) {
        const fp_instance& in = insts[build[k]];
        const int B = in.n_bases;
        const size_t o = pof[k];
        std::copy(in.base_lat, in.base_lat + B, hp + o);
        std::copy(in.pickup_lat, in.pickup_lat + M, hp + o + B);
        std::copy(in.delivery_lat, in.delivery_lat + M, hp + o + B + M);
        std::copy(in.base_lon, in.base_lon + B, hp + npts + o);
        std::copy(in.pickup_lon, in.pickup_lon + M, hp + npts + o + B);
        std::copy(in.delivery_lon, in.delivery_lon + M, hp + npts + o + B + M);
        const double* la = pts.p + o;
        const double* lo = pts.p + npts + o;
        const double* co = pts.p + 2 * npts + o;
        jobs[k] = fpk::TableJob{la, lo, co, la + B, lo + B, co + B, la + B + M, lo + B + M,
                                co + B + M, built.p + tof[k], B};
        dev[build[k]] = built.p + tof[k];
      });
      h2d(pts.p, hp, 2 * npts, st);
      d_jobs = DBuf<fpk::TableJob>(build.size(), st);
      h2d(d_jobs.p, jobs.data(), build.size(), st);
      check(fpk::launch_point_cos(pts.p, (int)npts, pts.p + 2 * npts, st), "cos(points)");
      check(fpk::launch_table_batch(d_jobs.p, (int)build.size(), M, maxB, radius_km, st),
            "table_batch");
      ctx->launches += 2;
    }
    run_search(ctx, n, insts, cfgs, starts, outs, dev, host);
  });
}

fp_status fp_search_batch(fp_ctx* ctx, int32_t n, const fp_instance* insts,
                          const double* const* tables, const fp_search_config* cfg,
                          const fp_search_start* starts, fp_search_result* outs) {
  if (n <= 0) return FP_OK;
  if (!cfg) return fail(FP_ERR_INVALID_ARGUMENT, "NULL search config");
  std::vector<fp_search_config> cfgs((size_t)n, *cfg);
  return fp_search_batch_configs(ctx, n, insts, tables, 6371.0088, cfgs.data(), starts, outs);
}

fp_status fp_neighbourhood_sweep(fp_ctx* ctx, const fp_instance* inst, const fp_search_start* start,
                                 fp_sweep_result* out) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!inst || !start || !out) throw FpError(FP_ERR_INVALID_ARGUMENT, "NULL argument");
    ensure_table(ctx, inst->n_missions, inst->n_bases);
    if (!ctx->table_ok)
      throw FpError(FP_ERR_INVALID_ARGUMENT,
                    "the sweep needs a distance table whose entries are finite and >= 0");
    // a local search's configuration: the sweep does not depend on it
    const fp_search_config cfg{0, FP_MODE_LOCAL, 0, -1, 0};
    fp_search_result r{};
    run_search(ctx, 1, inst, &cfg, start, &r, {ctx->d_cost}, {nullptr}, out);
  });
}

fp_status fp_enumerate_moves(fp_ctx* ctx, const fp_instance* in, const fp_search_start* state,
                             int32_t i, int32_t j, int32_t* out_kind, double* out_delta,
                             int32_t* out_count) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int M = in->n_missions, V = in->n_vehicles;
    ensure_table(ctx, M, in->n_bases);
    HostScenario h = prepare(in, state);
    if (j < 0 || j >= M) throw FpError(FP_ERR_ERROR, "unknown mission id");
    cudaStream_t st = ctx->stream;
    DBuf<int32_t> d_vb(V + 1), d_mv((size_t)M + 1);
    DBuf<double> d_out(4);
    h2d(d_vb.p, h.vbase.data(), V, st);
    h2d(d_mv.p, h.mv.data(), M, st);
    int n = 0;
    auto add = [&](int kind, int newcol, int mover) {
      check(fpk::launch_candidate_delta(ctx->d_cost, M, d_vb.p, d_mv.p, kind, j, newcol, mover,
                                        d_out.p + n, st),
            "candidate_delta");
      ctx->launches += 1;
      out_kind[n++] = kind;
    };
    const bool in_pool = i >= 0 && i < h.psize;
    // eval_takeover (search.cpp:82-101)
    if (in_pool && h.pkind[i] == fpk::POOL_IDLE) {
      const int g = h.pidx[i];
      if (!(in->rotary_only[j] && h.vfixed[g])) add(FP_MOVE_TAKEOVER, h.vbase[g], -1);
    }
    // eval_relocate (search.cpp:103-129)
    if (in_pool && h.pkind[i] == fpk::POOL_EMPTY) {
      const int t = h.pidx[i], mover = h.mv[j];
      if (!(h.vfixed[mover] && h.bheli[t])) add(FP_MOVE_RELOCATE, t, mover);
    }
    // eval_reassign (search.cpp:131-148)
    if (i >= 0 && i < M) {
      const int g = h.mv[i], l = h.mv[j];
      if (g != l && !(in->rotary_only[j] && h.vfixed[g])) add(FP_MOVE_REASSIGN, h.vbase[g], -1);
    }
    d2h(out_delta, d_out.p, n, st);
    check(cudaStreamSynchronize(st), "enumerate sync");
    *out_count = n;
  });
}

fp_status fp_objective_km(fp_ctx* ctx, int32_t n_vehicles, const int32_t* vehicle_base,
                          const int32_t* mission_vehicle, double* out_km) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->M < 0) throw FpError(FP_ERR_INVALID_ARGUMENT, "no resident table");
    const int M = ctx->M, V = n_vehicles;
    if (V < 0 || (V > 0 && !vehicle_base) || (M > 0 && !mission_vehicle) || !out_km)
      throw FpError(FP_ERR_INVALID_ARGUMENT, "bad objective arguments");
    // every mission served by a vehicle placed on a base of the table
    // (objective_km throws InfeasibleError otherwise, proj/src/model.cpp:178-181)
    for (int m = 0; m < M; ++m) {
      const int v = mission_vehicle[m];
      if (v < 0 || v >= V)
        throw FpError(FP_ERR_INFEASIBLE, "mission index " + std::to_string(m) + " is not served");
      if (vehicle_base[v] < 0 || vehicle_base[v] >= ctx->B)
        throw FpError(FP_ERR_INFEASIBLE, "service references unplaced vehicle index " + std::to_string(v));
    }
    cudaStream_t st = ctx->stream;
    DBuf<int32_t> d_vb(V + 1), d_mv((size_t)M + 1);
    DBuf<double> d_out(1);
    h2d(d_vb.p, vehicle_base, V, st);
    h2d(d_mv.p, mission_vehicle, M, st);
    check(fpk::launch_objective(ctx->d_cost, M, d_vb.p, d_mv.p, d_out.p, st), "objective");
    ctx->launches += 1;
    d2h(out_km, d_out.p, 1, st);
    check(cudaStreamSynchronize(st), "objective sync");
  });
}

}  // extern "C"
