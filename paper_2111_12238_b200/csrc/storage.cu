// storage.cu -- L0 storage conversions of make_state (kernels.hpp:429-495)
// done on the GPU: lower_triangle, to_csr (stable transpose), row views,
// diagonal positions, the DSCAL vector, and system interleaving.
//
// Layout decision (B200-first): the numeric arrays of `nsys` systems that
// share one sparsity pattern are stored interleaved, value[p * nsys + s], so a
// warp touching one nonzero for all systems reads one contiguous 8*nsys-byte
// segment and every x[j] gather fetches all systems' x_j in one sector run.
#include "common.cuh"
#include "internal.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace sfg {

thread_local int64_t* g_launch_counter = nullptr;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

int sm_count() {
  int dev = 0, sms = 0;
  SFG_CUDA(cudaGetDevice(&dev));
  SFG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

namespace {

inline unsigned grid_for(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * 32;
  if (g > cap)
    g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename T> struct TmpBuf {
  T* p = nullptr;
  cudaStream_t s;
  TmpBuf(int64_t n, cudaStream_t st) : s(st) {
    if (n > 0)
      SFG_CUDA(cudaMallocAsync(&p, sizeof(T) * (size_t)n, s));
  }
  ~TmpBuf() {
    if (p)
      cudaFreeAsync(p, s);
  }
};

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 62 && (1ll << b) <= maxval)
    ++b;
  return b;
}

__global__ void expand_major_kernel(const int32_t* __restrict__ ptr,
                                    int32_t nmajor, int32_t* __restrict__ maj) {
  // one warp per major index: coalesced writes for long segments
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t m = warp; m < nmajor; m += nwarps) {
    const int32_t b = ptr[m], e = ptr[m + 1];
    for (int32_t p = b + lane; p < e; p += 32)
      maj[p] = (int32_t)m;
  }
}

__global__ void iota_kernel(int32_t* __restrict__ a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src,
                                  const int32_t* __restrict__ perm, int64_t n,
                                  int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[perm[i]];
}

// out_ptr[i] = first position q with keys[q] >= i, for i in [0, nminor].
__global__ void ptr_from_sorted_kernel(const int32_t* __restrict__ keys,
                                       int64_t nnz, int32_t nminor,
                                       int32_t* __restrict__ out_ptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nminor;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < i)
        lo = mid + 1;
      else
        hi = mid;
    }
    out_ptr[i] = (int32_t)lo;
  }
}

__global__ void gather_values_kernel(const double* __restrict__ in,
                                     int64_t stride,
                                     const int32_t* __restrict__ perm,
                                     int64_t nnz, int32_t nsys,
                                     double* __restrict__ out) {
  const int64_t total = nnz * nsys;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = t / nsys;
    const int32_t s = (int32_t)(t - q * nsys);
    const int64_t src = perm ? perm[q] : q;
    out[t] = in[(int64_t)s * stride + src];
  }
}

// lower_triangle pass 1: per column, first entry with row >= col, count, and
// the reference's validity checks (matrix.hpp:106-123) as a min-key.
__global__ void lower_scan_kernel(const int32_t* __restrict__ colptr,
                                  const int32_t* __restrict__ rowidx,
                                  const double* __restrict__ vals,
                                  int64_t stride, int32_t nsys, int32_t n,
                                  int32_t* __restrict__ start,
                                  int32_t* __restrict__ cnt,
                                  unsigned long long* bad) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = colptr[j], e = colptr[j + 1];
    int32_t lo = b, hi = e;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (rowidx[mid] < j)
        lo = mid + 1;
      else
        hi = mid;
    }
    start[j] = lo;
    cnt[j] = e - lo;
    if (lo == e || rowidx[lo] != j) {
      atomicMin(bad, ((unsigned long long)j << 1) | 1ull); // missing
    } else {
      for (int32_t s = 0; s < nsys; ++s)
        if (vals[(int64_t)s * stride + lo] == 0.0) {
          atomicMin(bad, ((unsigned long long)j << 1)); // zero
          break;
        }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    cnt[n] = 0;
}

__global__ void lower_copy_kernel(const int32_t* __restrict__ rowidx,
                                  const int32_t* __restrict__ start,
                                  const int32_t* __restrict__ lptr, int32_t n,
                                  int32_t* __restrict__ lidx,
                                  int32_t* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    const int32_t b = lptr[j], e = lptr[j + 1], s0 = start[j];
    for (int32_t a = lane; a < e - b; a += 32) {
      lidx[b + a] = rowidx[s0 + a];
      src[b + a] = s0 + a;
    }
  }
}

__global__ void reverse_segments_kernel(const int32_t* __restrict__ ptr,
                                        const int32_t* __restrict__ idx,
                                        int32_t nseg, int32_t* __restrict__ out,
                                        int32_t* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t m = warp; m < nseg; m += nwarps) {
    const int32_t b = ptr[m], e = ptr[m + 1];
    for (int32_t k = lane; k < e - b; k += 32) {
      out[b + k] = idx[e - 1 - k];
      perm[b + k] = e - 1 - k;
    }
  }
}

__global__ void find_diag_kernel(const int32_t* __restrict__ rowptr,
                                 const int32_t* __restrict__ colidx, int32_t n,
                                 int32_t* __restrict__ diag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = rowptr[i], hi = rowptr[i + 1];
    const int32_t e = hi;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (colidx[mid] < i)
        lo = mid + 1;
      else
        hi = mid;
    }
    diag[i] = (lo < e && colidx[lo] == i) ? lo : -1;
  }
}

__global__ void dscal_vector_kernel(const int32_t* __restrict__ colptr,
                                    const double* __restrict__ vals, int32_t n,
                                    double* __restrict__ d) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    d[j] = __ddiv_rn(1.0, __dsqrt_rn(fabs(vals[colptr[j]])));
}

__global__ void scaling_csr_kernel(const int32_t* __restrict__ diag,
                                   const double* __restrict__ vals, int32_t n,
                                   double* __restrict__ d, int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = diag[i] >= 0 ? vals[diag[i]] : 0.0;
    if (a == 0.0)
      atomicMin(bad, (int)i);
    d[i] = __ddiv_rn(1.0, __dsqrt_rn(fabs(a)));
  }
}

__global__ void interleave_kernel(const double* __restrict__ in, int32_t n,
                                  int32_t nsys, double* __restrict__ out,
                                  int to_inter) {
  const int64_t total = (int64_t)n * nsys;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nsys;
    const int32_t s = (int32_t)(t - i * nsys);
    if (to_inter)
      out[t] = in[(int64_t)s * n + i];
    else
      out[(int64_t)s * n + i] = in[t];
  }
}

} // namespace

void transpose(const int32_t* ptr, const int32_t* idx, int32_t nmajor,
               int32_t nminor, int64_t nnz, int32_t* out_ptr, int32_t* out_idx,
               int32_t* perm, cudaStream_t s) {
  if (nnz == 0) {
    SFG_CUDA(cudaMemsetAsync(out_ptr, 0, sizeof(int32_t) * ((size_t)nminor + 1), s));
    return;
  }
  TmpBuf<int32_t> maj(nnz, s), iota(nnz, s), keys_out(nnz, s);
  expand_major_kernel<<<grid_for((int64_t)nmajor * 32), 256, 0, s>>>(ptr, nmajor, maj.p);
  iota_kernel<<<grid_for(nnz), 256, 0, s>>>(iota.p, nnz);
  count_launch(2);
  size_t tmp_bytes = 0;
  const int end_bit = bits_for(nminor);
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, idx, keys_out.p,
                                           iota.p, perm, (int)nnz, 0, end_bit, s));
  TmpBuf<char> tmp((int64_t)tmp_bytes, s);
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, idx, keys_out.p,
                                           iota.p, perm, (int)nnz, 0, end_bit, s));
  gather_i32_kernel<<<grid_for(nnz), 256, 0, s>>>(maj.p, perm, nnz, out_idx);
  ptr_from_sorted_kernel<<<grid_for((int64_t)nminor + 1), 256, 0, s>>>(
      keys_out.p, nnz, nminor, out_ptr);
  count_launch(3);
  SFG_CUDA(cudaGetLastError());
}

void gather_values(const double* in, int64_t in_stride, const int32_t* perm,
                   int64_t nnz, int32_t nsys, double* out, cudaStream_t s) {
  if (nnz == 0)
    return;
  gather_values_kernel<<<grid_for(nnz * nsys), 256, 0, s>>>(in, in_stride, perm,
                                                            nnz, nsys, out);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

int64_t lower_triangle(const int32_t* colptr, const int32_t* rowidx,
                       const double* vals, int64_t val_stride, int32_t nsys,
                       int32_t n, DBuf<int32_t>& lptr, DBuf<int32_t>& lidx,
                       DBuf<int32_t>& src_pos, cudaStream_t s) {
  TmpBuf<int32_t> start(n + 1, s), cnt(n + 1, s);
  TmpBuf<unsigned long long> bad(1, s);
  SFG_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
  lower_scan_kernel<<<grid_for(n), 256, 0, s>>>(colptr, rowidx, vals, val_stride,
                                                nsys, n, start.p, cnt.p, bad.p);
  count_launch();
  lptr.alloc((int64_t)n + 1);
  size_t tmp_bytes = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, lptr.p, n + 1, s));
  TmpBuf<char> tmp((int64_t)tmp_bytes, s);
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, lptr.p, n + 1, s));
  unsigned long long hbad = 0;
  int32_t lnnz = 0;
  SFG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(hbad), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaMemcpyAsync(&lnnz, lptr.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    const int32_t j = (int32_t)(hbad >> 1);
    if (hbad & 1ull)
      throw InvalidMatrix("missing diagonal entry at column " + std::to_string(j), j);
    throw InvalidMatrix("zero diagonal entry at column " + std::to_string(j), j);
  }
  lidx.alloc(lnnz);
  src_pos.alloc(lnnz);
  lower_copy_kernel<<<grid_for((int64_t)n * 32), 256, 0, s>>>(rowidx, start.p, lptr.p,
                                                              n, lidx.p, src_pos.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  return lnnz;
}

void reverse_segments(const int32_t* ptr, const int32_t* idx, int32_t nseg,
                      int32_t* out_idx, int32_t* perm, cudaStream_t s) {
  reverse_segments_kernel<<<grid_for((int64_t)nseg * 32), 256, 0, s>>>(ptr, idx, nseg,
                                                                       out_idx, perm);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void find_diag_positions(const int32_t* rowptr, const int32_t* colidx,
                         int32_t n, int32_t* diag, cudaStream_t s) {
  find_diag_kernel<<<grid_for(n), 256, 0, s>>>(rowptr, colidx, n, diag);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

int32_t scaling_vector_csr(const int32_t* diag, const double* vals, int32_t n, double* d,
                           cudaStream_t s) {
  if (n == 0)
    return -1;
  int* bad = nullptr;
  SFG_CUDA(cudaMallocAsync(&bad, sizeof(int), s));
  const int init = 0x7fffffff;
  SFG_CUDA(cudaMemcpyAsync(bad, &init, sizeof(int), cudaMemcpyHostToDevice, s));
  scaling_csr_kernel<<<grid_for(n), 256, 0, s>>>(diag, vals, n, d, bad);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  int h = init;
  SFG_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaFreeAsync(bad, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  return h == init ? -1 : h;
}

void dscal_vector(const int32_t* colptr, const double* vals, int32_t n,
                  double* d, cudaStream_t s) {
  dscal_vector_kernel<<<grid_for(n), 256, 0, s>>>(colptr, vals, n, d);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void interleave(const double* sys_major, int32_t n, int32_t nsys, double* inter,
                cudaStream_t s) {
  if (nsys == 1) {
    SFG_CUDA(cudaMemcpyAsync(inter, sys_major, sizeof(double) * (size_t)n,
                             cudaMemcpyDeviceToDevice, s));
    return;
  }
  interleave_kernel<<<grid_for((int64_t)n * nsys), 256, 0, s>>>(sys_major, n, nsys,
                                                               inter, 1);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void deinterleave(const double* inter, int32_t n, int32_t nsys,
                  double* sys_major, cudaStream_t s) {
  if (nsys == 1) {
    SFG_CUDA(cudaMemcpyAsync(sys_major, inter, sizeof(double) * (size_t)n,
                             cudaMemcpyDeviceToDevice, s));
    return;
  }
  interleave_kernel<<<grid_for((int64_t)n * nsys), 256, 0, s>>>(inter, n, nsys,
                                                               sys_major, 0);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

} // namespace sfg
