// pcg.cu -- preconditioned conjugate gradients on the GPU with the fused
// executors as its preconditioner (SURVEY 8f "next" 3: the iterative solver
// that repeats the executor and so amortises the inspector; PAPER.md:948 --
// SpTRSV pairs are the main bottleneck of preconditioned CG).
//
// Setup: a combo-5 plan on A produces the IC0 factor L (ic0_column,
// kernels.hpp:214-242, bit-exact); a combo-8 plan on L's pattern applies
// M^-1 r = L^-T (L^-1 r) -- the fused forward/backward pair of BASELINE
// config 5.  Each iteration: q = A p with the dot p.q, the x / r updates with
// r.r, the preconditioner, r.z, and p = z + beta p.  Reductions are
// two-pass (per-block partials summed in block order by one block), so a
// solve is deterministic run to run.  Scalars stay on the device; the host
// reads the residual once per `check` iterations.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "../../include/sfgpu.h"

struct sfg_pcg {
  int device = 0;
  int32_t n = 0;
  cudaStream_t stream = nullptr;
  sfg_plan* fac = nullptr; // combo 5 on A: the IC0 factor
  sfg_plan* sol = nullptr; // combo 8 on L: the preconditioner apply
  sfg::DBuf<int32_t> a_ptr, a_idx; // A in CSR for the SpMV
  sfg::DBuf<double> a_val;
  sfg::DBuf<double> x, r, z, p, q, part;
  sfg::DBuf<double> scal; // [0] p.q  [1] r.r  [2] r.z (old)  [3] r.z (new)  [4] b.b
  double* host_scal = nullptr;
  int64_t nnzL = 0;
  std::vector<int32_t> l_ptr, l_idx; // host pattern of L (for the combo-8 plan)
};

namespace {

constexpr int kT = 256;
constexpr int kMaxBlocks = 1024; // partial sums per reduction

int blocks_for(int32_t n) {
  int b = (n + kT - 1) / kT;
  return b < 1 ? 1 : (b > kMaxBlocks ? kMaxBlocks : b);
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0)
    sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kT / 32; ++w)
      t += sh[w];
  return t;
}

// q = A p (CSR rows, ascending columns) and per-block partials of p.q
__global__ void k_spmv_dot(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                           const double* __restrict__ val, const double* __restrict__ p,
                           double* __restrict__ q, int32_t n, double* __restrict__ part) {
  double acc = 0.0;
  for (int32_t i = blockIdx.x * kT + threadIdx.x; i < n; i += gridDim.x * kT) {
    double s = 0.0;
    for (int32_t e = ptr[i]; e < ptr[i + 1]; ++e)
      s = fma(val[e], p[idx[e]], s);
    q[i] = s;
    acc = fma(p[i], s, acc);
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0)
    part[blockIdx.x] = t;
}

// per-block partials of a.b
__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int32_t n,
                      double* __restrict__ part) {
  double acc = 0.0;
  for (int32_t i = blockIdx.x * kT + threadIdx.x; i < n; i += gridDim.x * kT)
    acc = fma(a[i], b[i], acc);
  const double t = block_sum(acc);
  if (threadIdx.x == 0)
    part[blockIdx.x] = t;
}

// one block: out = sum of nb partials in block order
__global__ void k_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += kT)
    acc += part[i];
  const double t = block_sum(acc);
  if (threadIdx.x == 0)
    *out = t;
}

// alpha = rz / pq; x += alpha p; r -= alpha q; partials of r.r
__global__ void k_update_xr(double* __restrict__ x, double* __restrict__ r,
                            const double* __restrict__ p, const double* __restrict__ q, int32_t n,
                            const double* __restrict__ scal, double* __restrict__ part) {
  const double alpha = scal[2] / scal[0];
  double acc = 0.0;
  for (int32_t i = blockIdx.x * kT + threadIdx.x; i < n; i += gridDim.x * kT) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    acc = fma(ri, ri, acc);
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0)
    part[blockIdx.x] = t;
}

// beta = rz_new / rz_old; p = z + beta p  (first = true: p = z)
__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ z, int32_t n,
                           const double* __restrict__ scal, int first) {
  const double beta = first ? 0.0 : scal[3] / scal[2];
  for (int32_t i = blockIdx.x * kT + threadIdx.x; i < n; i += gridDim.x * kT)
    p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}

__global__ void k_shift_rz(double* scal) { scal[2] = scal[3]; }

void launched() { sfg::count_launch(); }

void dot_into(sfg_pcg* S, const double* a, const double* b, double* out) {
  const int nb = blocks_for(S->n);
  k_dot<<<nb, kT, 0, S->stream>>>(a, b, S->n, S->part.p);
  k_final<<<1, kT, 0, S->stream>>>(S->part.p, nb, out);
  launched();
  launched();
}

sfg_status apply_precond(sfg_pcg* S) { // z = L^-T L^-1 r
  sfg_status st = sfg_set_vin_device(S->sol, S->r.p);
  if (st == SFG_OK)
    st = sfg_execute_fused(S->sol);
  if (st != SFG_OK)
    return st;
  void* vout = nullptr;
  int64_t cnt = 0;
  st = sfg_device_output(S->sol, 1, &vout, &cnt);
  if (st != SFG_OK)
    return st;
  SFG_CUDA(cudaMemcpyAsync(S->z.p, vout, sizeof(double) * (size_t)S->n, cudaMemcpyDeviceToDevice,
                           S->stream));
  return SFG_OK;
}

} // namespace

extern "C" {

sfg_status sfg_pcg_create(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                          const double* values, sfg_pcg** out) {
  if (!out || n < 0 || !colptr)
    return SFG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
    cudaGetLastError();
    return SFG_ERR_NO_DEVICE;
  }
  auto* S = new sfg_pcg();
  S->n = n;
  cudaGetDevice(&S->device);
  try {
    SFG_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
    // IC0 factor of A (combo 5; its solve output is not used)
    sfg_status st = sfg_plan_create(5, n, colptr, rowidx, values, 1, nullptr, 7, &S->fac);
    if (st != SFG_OK) {
      *out = S;
      return st;
    }
    sfg_plan_set_stream(S->fac, S->stream);
    if ((st = sfg_inspect(S->fac)) != SFG_OK || (st = sfg_execute_fused(S->fac)) != SFG_OK ||
        (st = sfg_synchronize(S->fac)) != SFG_OK) {
      *out = S;
      return st;
    }
    // L's pattern (lower triangle of A, CSC, diagonal first) and values
    S->l_ptr.assign((size_t)n + 1, 0);
    for (int32_t j = 0; j < n; ++j) {
      int32_t c = 0;
      for (int32_t e = colptr[j]; e < colptr[j + 1]; ++e)
        c += rowidx[e] >= j ? 1 : 0;
      S->l_ptr[(size_t)j + 1] = S->l_ptr[(size_t)j] + c;
    }
    S->nnzL = S->l_ptr[(size_t)n];
    S->l_idx.resize((size_t)S->nnzL);
    for (int32_t j = 0, w = 0; j < n; ++j)
      for (int32_t e = colptr[j]; e < colptr[j + 1]; ++e)
        if (rowidx[e] >= j)
          S->l_idx[(size_t)w++] = rowidx[e];
    std::vector<double> lval((size_t)S->nnzL);
    if (S->nnzL) {
      void* fac = nullptr;
      int64_t fc = 0;
      sfg_device_output(S->fac, 0, &fac, &fc);
      SFG_CUDA(cudaMemcpy(lval.data(), fac, sizeof(double) * (size_t)S->nnzL,
                          cudaMemcpyDeviceToHost));
    }
    st = sfg_plan_create(8, n, S->l_ptr.data(), S->l_idx.data(), lval.data(), 1, nullptr, 7,
                         &S->sol);
    if (st != SFG_OK) {
      *out = S;
      return st;
    }
    sfg_plan_set_stream(S->sol, S->stream);
    if ((st = sfg_inspect(S->sol)) != SFG_OK) {
      *out = S;
      return st;
    }
    // A in CSR for the SpMV
    const int32_t nnz = colptr[n];
    std::vector<int32_t> rp((size_t)n + 1, 0), ci((size_t)nnz);
    std::vector<double> cv((size_t)nnz);
    for (int32_t e = 0; e < nnz; ++e)
      ++rp[(size_t)rowidx[e] + 1];
    for (int32_t i = 0; i < n; ++i)
      rp[(size_t)i + 1] += rp[(size_t)i];
    std::vector<int32_t> cur(rp.begin(), rp.end() - 1);
    for (int32_t j = 0; j < n; ++j)
      for (int32_t e = colptr[j]; e < colptr[j + 1]; ++e) {
        const int32_t w = cur[(size_t)rowidx[e]]++;
        ci[(size_t)w] = j;
        cv[(size_t)w] = values[e];
      }
    S->a_ptr.alloc((int64_t)n + 1);
    S->a_idx.alloc(nnz > 0 ? nnz : 1);
    S->a_val.alloc(nnz > 0 ? nnz : 1);
    SFG_CUDA(cudaMemcpy(S->a_ptr.p, rp.data(), sizeof(int32_t) * rp.size(), cudaMemcpyHostToDevice));
    if (nnz) {
      SFG_CUDA(cudaMemcpy(S->a_idx.p, ci.data(), sizeof(int32_t) * ci.size(), cudaMemcpyHostToDevice));
      SFG_CUDA(cudaMemcpy(S->a_val.p, cv.data(), sizeof(double) * cv.size(), cudaMemcpyHostToDevice));
    }
    const int64_t nn = n > 0 ? n : 1;
    S->x.alloc(nn);
    S->r.alloc(nn);
    S->z.alloc(nn);
    S->p.alloc(nn);
    S->q.alloc(nn);
    S->part.alloc(kMaxBlocks);
    S->scal.alloc(8);
    SFG_CUDA(cudaHostAlloc(&S->host_scal, sizeof(double) * 8, cudaHostAllocDefault));
  } catch (const std::exception&) {
    *out = S;
    return SFG_ERR_CUDA;
  }
  *out = S;
  return SFG_OK;
}

sfg_status sfg_pcg_solve(sfg_pcg* S, const double* b_host, double* x_host, double rtol,
                         int32_t maxit, int32_t check, int32_t* iters, double* relres,
                         float* ms) {
  if (!S || !S->sol || !b_host || !x_host || maxit < 0)
    return SFG_ERR_INVALID_ARGUMENT;
  if (check < 1)
    check = 1;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != S->device)
    cudaSetDevice(S->device);
  sfg_status result = SFG_OK;
  try {
    const int32_t n = S->n;
    const int nb = blocks_for(n);
    cudaEvent_t e0, e1;
    SFG_CUDA(cudaEventCreate(&e0));
    SFG_CUDA(cudaEventCreate(&e1));
    SFG_CUDA(cudaMemcpyAsync(S->r.p, b_host, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice,
                             S->stream));
    SFG_CUDA(cudaEventRecord(e0, S->stream));
    SFG_CUDA(cudaMemsetAsync(S->x.p, 0, sizeof(double) * (size_t)n, S->stream));
    SFG_CUDA(cudaMemsetAsync(S->scal.p, 0, sizeof(double) * 8, S->stream));
    dot_into(S, S->r.p, S->r.p, S->scal.p + 4); // b.b
    if ((result = apply_precond(S)) != SFG_OK)
      throw std::runtime_error("precond");
    dot_into(S, S->r.p, S->z.p, S->scal.p + 2); // r.z
    k_update_p<<<nb, kT, 0, S->stream>>>(S->p.p, S->z.p, n, S->scal.p, 1);
    launched();
    SFG_CUDA(cudaMemcpyAsync(S->host_scal, S->scal.p, sizeof(double) * 8, cudaMemcpyDeviceToHost,
                             S->stream));
    SFG_CUDA(cudaStreamSynchronize(S->stream));
    const double bnorm = std::sqrt(S->host_scal[4]);
    int32_t it = 0;
    double rel = bnorm > 0.0 ? 1.0 : 0.0;
    while (it < maxit && rel > rtol) {
      k_spmv_dot<<<nb, kT, 0, S->stream>>>(S->a_ptr.p, S->a_idx.p, S->a_val.p, S->p.p, S->q.p, n,
                                          S->part.p);
      k_final<<<1, kT, 0, S->stream>>>(S->part.p, nb, S->scal.p + 0); // p.q
      k_update_xr<<<nb, kT, 0, S->stream>>>(S->x.p, S->r.p, S->p.p, S->q.p, n, S->scal.p,
                                           S->part.p);
      k_final<<<1, kT, 0, S->stream>>>(S->part.p, nb, S->scal.p + 1); // r.r
      for (int k = 0; k < 4; ++k)
        launched();
      ++it;
      if (it % check == 0 || it == maxit) {
        SFG_CUDA(cudaMemcpyAsync(S->host_scal, S->scal.p, sizeof(double) * 8,
                                 cudaMemcpyDeviceToHost, S->stream));
        SFG_CUDA(cudaStreamSynchronize(S->stream));
        rel = bnorm > 0.0 ? std::sqrt(S->host_scal[1]) / bnorm : 0.0;
        if (rel <= rtol || !(rel == rel))
          break;
      }
      if ((result = apply_precond(S)) != SFG_OK)
        throw std::runtime_error("precond");
      dot_into(S, S->r.p, S->z.p, S->scal.p + 3); // r.z (new)
      k_update_p<<<nb, kT, 0, S->stream>>>(S->p.p, S->z.p, n, S->scal.p, 0);
      k_shift_rz<<<1, 1, 0, S->stream>>>(S->scal.p);
      launched();
      launched();
    }
    SFG_CUDA(cudaEventRecord(e1, S->stream));
    SFG_CUDA(cudaMemcpyAsync(x_host, S->x.p, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost,
                             S->stream));
    SFG_CUDA(cudaMemcpyAsync(S->host_scal, S->scal.p, sizeof(double) * 8, cudaMemcpyDeviceToHost,
                             S->stream));
    SFG_CUDA(cudaStreamSynchronize(S->stream));
    rel = bnorm > 0.0 ? std::sqrt(S->host_scal[1]) / bnorm : 0.0;
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (iters)
      *iters = it;
    if (relres)
      *relres = it == 0 ? (bnorm > 0.0 ? 1.0 : 0.0) : rel;
    if (ms)
      *ms = t;
  } catch (const std::exception&) {
    if (result == SFG_OK)
      result = SFG_ERR_CUDA;
  }
  if (prev != S->device)
    cudaSetDevice(prev);
  return result;
}

sfg_status sfg_pcg_plans(const sfg_pcg* S, sfg_plan** factor_plan, sfg_plan** solve_plan) {
  if (!S)
    return SFG_ERR_INVALID_ARGUMENT;
  if (factor_plan)
    *factor_plan = S->fac;
  if (solve_plan)
    *solve_plan = S->sol;
  return SFG_OK;
}

sfg_status sfg_pcg_destroy(sfg_pcg* S) {
  if (!S)
    return SFG_OK;
  cudaSetDevice(S->device);
  if (S->stream)
    cudaStreamSynchronize(S->stream);
  if (S->fac)
    sfg_plan_destroy(S->fac);
  if (S->sol)
    sfg_plan_destroy(S->sol);
  if (S->host_scal)
    cudaFreeHost(S->host_scal);
  S->a_ptr.release();
  S->a_idx.release();
  S->a_val.release();
  S->x.release();
  S->r.release();
  S->z.release();
  S->p.release();
  S->q.release();
  S->part.release();
  S->scal.release();
  if (S->stream)
    cudaStreamDestroy(S->stream);
  delete S;
  return SFG_OK;
}

} // extern "C"
