// perm_kernels.cu — the search's permutation stream on the device.
//
// tabu_search draws perm_a and perm_b of every pass from one std::mt19937_64
// seeded with SearchConfig::seed (proj/src/search.cpp:401-413, SURVEY.md §8a
// T11): Fisher–Yates from i = n down to 2 with j = uniform_below(i), where
// uniform_below rejects draws below (2^64 - i) mod i. The host generator of
// api.cpp (PermStream) reproduces that stream; for batches it is the
// bottleneck (one sequential stream, ~10 ns per draw), so here:
//  * mt_gen_kernel: one block runs the generator's sequential part — the
//    312-word twist in two data-parallel phases (the in-place sequential
//    update reads old words ahead of i and new words behind it) — and stores
//    the raw state words;
//  * fy_kernel: block per permutation — the tempering of its draws and
//    j = x mod i for every step in parallel, then the sequential swaps in
//    shared memory by one thread.
// A permutation consumes exactly n - 1 draws unless a draw is rejected
// (probability ~ n / 2^64 per draw); a rejection is flagged, the pass kernels
// refuse to run on the chunk, and the host regenerates the stream exactly.

#include <cstdint>

#include "common.cuh"

namespace fpk {

namespace {

constexpr unsigned long long kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;
constexpr unsigned long long kMatrixA = 0xB5026F5AA96619E9ull;

__device__ __forceinline__ unsigned long long twist_word(unsigned long long a, unsigned long long b,
                                                         unsigned long long c) {
  const unsigned long long y = (a & kUpper) | (b & kLower);
  return c ^ (y >> 1) ^ ((y & 1ull) ? kMatrixA : 0ull);
}

__device__ __forceinline__ unsigned long long temper(unsigned long long x) {
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

}  // namespace

// Appends `count` outputs of the generator held in st[blockIdx.x] to
// out + blockIdx.x * count, UNTEMPERED (the consumer applies temper()). One
// block of 320 threads per stream. The state is double-buffered in shared
// memory (round r reads buffer r&1 and writes the other), so a round is two
// barriers: phase A (k < 156: old words only), phase B (k >= 156: old words
// and phase A's new ones); the stores of a round overlap the next round's
// phase A. The tempering (half of the per-output work) is left to the
// parallel consumer, off the generator's sequential critical path.
__global__ void __launch_bounds__(320) mt_gen_kernel(MtState* st, unsigned long long* out,
                                                     long long count) {
  __shared__ unsigned long long mt[2][312];
  st += blockIdx.x;
  out += (long long)blockIdx.x * count;
  const int t = threadIdx.x;
  for (int k = t; k < 312; k += blockDim.x) mt[0][k] = st->mt[k];
  int idx = st->idx;
  int cur = 0;  // the buffer holding the current state
  __syncthreads();
  long long produced = 0;
  // the rest of the current state's outputs
  if (idx < 312) {
    const int n = (int)min((long long)(312 - idx), count);
    if (t < n) out[t] = mt[cur][idx + t];
    idx += n;
    produced += n;
  }
  while (produced < count) {
    const unsigned long long* o = mt[cur];
    unsigned long long* w = mt[cur ^ 1];
    // phase A: k < 156 reads old k, k+1, k+156
    if (t < 156) w[t] = twist_word(o[t], o[t + 1], o[t + 156]);
    __syncthreads();
    // phase B: 156 <= k < 312 reads old k, k+1 (k = 311: new 0) and new k-156
    if (t >= 156 && t < 312) w[t] = twist_word(o[t], t == 311 ? w[0] : o[t + 1], w[t - 156]);
    __syncthreads();
    cur ^= 1;
    const int n = (int)min(312ll, count - produced);
    if (t < n) out[produced + t] = mt[cur][t];
    idx = n;
    produced += n;
  }
  __syncthreads();
  for (int k = t; k < 312; k += blockDim.x) st->mt[k] = mt[cur][k];
  if (t == 0) st->idx = idx;
}

// Permutation p of nperm (n elements) from draws[p*(n-1) ...] (untempered
// state words: x = temper(word)): Fisher–Yates with j_i = x mod i. Dynamic
// shared memory: 4*(2n+1) bytes.
__global__ void __launch_bounds__(256) fy_kernel(const unsigned long long* __restrict__ draws, int n,
                                                 int32_t* __restrict__ perms, int* bad) {
  extern __shared__ int fy_smem[];
  int* out = fy_smem;      // [n]
  int* jv = fy_smem + n;   // [n + 1], jv[i] for i = 2..n
  const long long base = (long long)blockIdx.x * (n - 1);
  for (int i = 2 + threadIdx.x; i <= n; i += blockDim.x) {
    const unsigned long long x = temper(draws[base + (n - i)]);
    const unsigned long long ui = (unsigned long long)i;
    if (x < (0ull - ui) % ui) atomicOr(bad, 1);
    jv[i] = (int)(x % ui);
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = n; i > 1; --i) {
      const int j = jv[i];
      const int a = out[i - 1];
      out[i - 1] = out[j];
      out[j] = a;
    }
  }
  __syncthreads();
  int32_t* dst = perms + (long long)blockIdx.x * n;
  for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = out[k];
}

// The seeded states (std::mersenne_twister_engine::seed) on the device: the
// search's first permutation chunk needs no host copy in front of it.
__global__ void mt_seed_kernel(MtState* st, MtSeeds seeds, int n) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  unsigned long long x = seeds.seed[d];
  st[d].mt[0] = x;
  for (int i = 1; i < 312; ++i) {
    x = 6364136223846793005ull * (x ^ (x >> 62)) + (unsigned)i;
    st[d].mt[i] = x;
  }
  st[d].idx = 312;
}

cudaError_t launch_mt_seed(MtState* st, const unsigned long long* seeds, int n, cudaStream_t stream) {
  for (int d0 = 0; d0 < n; d0 += MtSeeds::kMax) {
    MtSeeds b;
    const int k = n - d0 < MtSeeds::kMax ? n - d0 : MtSeeds::kMax;
    for (int i = 0; i < k; ++i) b.seed[i] = seeds[d0 + i];
    mt_seed_kernel<<<1, MtSeeds::kMax, 0, stream>>>(st + d0, b, k);
  }
  return cudaGetLastError();
}

// Host: the seeded state (std::mersenne_twister_engine::seed).
void mt_seed_host(MtState* st, unsigned long long seed) {
  st->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    st->mt[i] = 6364136223846793005ull * (st->mt[i - 1] ^ (st->mt[i - 1] >> 62)) + (unsigned)i;
  st->idx = 312;
}

size_t fy_smem_bytes(int n) { return sizeof(int) * (2ull * n + 1); }

// For each of `nstreams` independent streams (states st[0..nstreams)),
// nperm permutations of n (n >= 2) continuing that stream, written stream
// after stream: perms[(d * nperm + p) * n ...]. draws is scratch of
// nstreams * nperm * (n - 1) words.
cudaError_t launch_permutations(MtState* st, int nstreams, int n, int nperm,
                                unsigned long long* draws, int32_t* perms, int* bad,
                                cudaStream_t stream) {
  if (nperm <= 0 || nstreams <= 0) return cudaSuccess;
  mt_gen_kernel<<<nstreams, 320, 0, stream>>>(st, draws, (long long)nperm * (n - 1));
  const size_t smem = fy_smem_bytes(n);
  cudaFuncSetAttribute(fy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fy_kernel<<<nstreams * nperm, 256, smem, stream>>>(draws, n, perms, bad);
  return cudaGetLastError();
}

}  // namespace fpk
