// host_common.hpp — host-side error plumbing and kernel launcher prototypes.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "fleetplace_b200.h"

namespace fpk {
struct Scenario;
struct MtState;

void mt_seed_host(MtState* st, unsigned long long seed);
cudaError_t launch_mt_seed(MtState* st, const unsigned long long* seeds, int n, cudaStream_t stream);
size_t fy_smem_bytes(int n);
cudaError_t launch_permutations(MtState* st, int nstreams, int n, int nperm,
                                unsigned long long* draws, int32_t* perms, int* bad,
                                cudaStream_t stream);
cudaError_t launch_table_check(const double* t, size_t n, int* bad, cudaStream_t st);
cudaError_t launch_table_check_multi(const double* const* d_ptrs, const long long* d_ns, int count,
                                     long long max_n, int* d_bad, cudaStream_t st);
struct TableJob;
cudaError_t launch_table_batch(const TableJob* d_jobs, int n_jobs, int M, int max_B,
                               double radius_km, cudaStream_t st);

void keep_pool_mapped(int dev);
cudaError_t launch_point_cos(const double* lat, int n, double* out, cudaStream_t st);
cudaError_t launch_transpose(const double* src, int M, int B, double* dst, cudaStream_t stream);
cudaError_t launch_table(const double* blat, const double* blon, const double* bcos, int B,
                         const double* plat, const double* plon, const double* pcos,
                         const double* dlat, const double* dlon, const double* dcos, int M,
                         double radius_km, double* cost, cudaStream_t st);
cudaError_t launch_table_auto(const double* blat, const double* blon, const double* bcos, int B,
                              const double* plat, const double* plon, const double* pcos,
                              const double* dlat, const double* dlon, const double* dcos, int M,
                              double radius_km, double* cost, cudaStream_t st, int* used_sites);
cudaError_t launch_haversine_pairs(int n, const double* alat, const double* alon,
                                   const double* blat, const double* blon, const double* clat,
                                   const double* clon, double radius_km, double* out,
                                   cudaStream_t st);
cudaError_t launch_column_totals(const double* cost, int M, int B, double* out, cudaStream_t st);
cudaError_t launch_column_totals_chain(const double* cost, int M, int B, const double* carry,
                                       double* out, cudaStream_t st);
cudaError_t launch_mission_argmin(const double* cost, int M, const int32_t* cb, const int32_t* cbid,
                                  const uint8_t* cf, const int32_t* cv, int n, const uint8_t* ro,
                                  int32_t* mv, int32_t* first_bad, cudaStream_t st);
cudaError_t launch_objective(const double* cost, int M, const int32_t* vb, const int32_t* mv,
                             double* out, cudaStream_t st);
cudaError_t launch_candidate_delta(const double* cost, int M, const int32_t* vb, const int32_t* mv,
                                   int kind, int j, int newcol, int mover, double* out,
                                   cudaStream_t st);
cudaError_t launch_init(Scenario* d_scs, const Scenario* h_scs, int n_scn, int M, int maxB,
                        int maxV, bool transpose, cudaStream_t stream, cudaEvent_t* ev,
                        bool exact_total = true, cudaStream_t side = nullptr);
cudaError_t launch_final(Scenario* d_scs, int n_scn, cudaStream_t stream);
cudaError_t launch_gather_results(const Scenario* d_scs, int n_scn, int M, int32_t* out_mv,
                                  int32_t* out_vb, const long long* vb_off, cudaStream_t stream);
cudaError_t launch_sweep(Scenario* d_scs, const int32_t* d_active, int n_scn,
                         const int32_t* d_perms, int M, cudaStream_t stream);
cudaError_t launch_pass(Scenario* d_scs, const int32_t* d_active, int n_scn,
                        const int32_t* d_perms, int kpasses, bool inkernel, int max_passes, int M,
                        bool tabu, long long tenure, bool debug, int V, int B, int K,
                        cudaStream_t stream, int threads, int helpers_req, unsigned epoch,
                        const int* perm_bad, bool global_bits = false);
}  // namespace fpk

namespace fpk_host {

// An fp_status carried through C++ code up to the C boundary.
struct FpError : std::runtime_error {
  FpError(fp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
  fp_status code;
};

struct CudaError : FpError {
  CudaError(cudaError_t e, const char* what)
      : FpError(e == cudaErrorMemoryAllocation ? FP_ERR_OUT_OF_MEMORY : FP_ERR_CUDA,
                std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what) {}
};

}  // namespace fpk_host
