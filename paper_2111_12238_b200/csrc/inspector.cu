// inspector.cu -- the inspector on the GPU (replaces make_dag / level_info /
// build_wavefront_schedule, dag.hpp:52-69,197-218, executor.hpp:209-229).
//
// * DAG CSR construction: edges become 64-bit (u << 32 | v) keys; one radix
//   sort + unique reproduces make_dag's "sort, unique, bucket by source".
// * Levels: level[v] = 1 + max(level[u]) is a triangular solve in the
//   (max, +) semiring, run with the same sync-free machinery as the executor:
//   ascending tickets, each vertex polls its predecessors' level words.
// * Heights: the same over successors with descending tickets.
// * Wavefront order: a stable radix sort of vertices by level (ascending
//   vertex id inside a level, as executor.hpp:215-217).
#include "common.cuh"
#include "internal.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>

namespace sfg {

namespace {

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

inline unsigned grid_for(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * 32;
  if (g > cap)
    g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

__global__ void ptr_from_keys_kernel(const uint64_t* __restrict__ keys,
                                     int64_t ne, int32_t nvert,
                                     int32_t* __restrict__ ptr,
                                     int32_t* __restrict__ idx) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u = tid; u <= nvert; u += stride) {
    const uint64_t key = (uint64_t)u << 32;
    int64_t lo = 0, hi = ne;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    ptr[u] = (int32_t)lo;
  }
  for (int64_t e = tid; e < ne; e += stride)
    idx[e] = (int32_t)(keys[e] & 0xffffffffull);
}

__global__ void flip_keys_kernel(const int32_t* __restrict__ ptr,
                                 const int32_t* __restrict__ idx, int32_t nvert,
                                 uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < nvert; u += nwarps)
    for (int32_t p = ptr[u] + lane; p < ptr[u + 1]; p += 32)
      keys[p] = ((uint64_t)(uint32_t)idx[p] << 32) | (uint32_t)u;
}

__global__ void levels_kernel(const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ idx, int32_t nvert,
                              int dir, int* level,
                              unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const long long base = claim_tickets(counter, 32);
    if (base >= nvert)
      break;
    const long long t = base + lane;
    if (t >= nvert)
      continue;
    const int v = dir > 0 ? (int)t : nvert - 1 - (int)t;
    int lv = 1;
    for (int p = __ldg(ptr + v); p < __ldg(ptr + v + 1); ++p) {
      const int u = __ldg(idx + p);
      if (dir > 0 ? (u < v) : (u > v)) {
        const int lu = poll_pos_i32(level + u) + 1;
        lv = lu > lv ? lu : lv;
      }
    }
    st_relaxed_i32(level + v, lv);
  }
}

__global__ void heights_kernel(const int32_t* __restrict__ succptr,
                               const int32_t* __restrict__ succ, int32_t nvert,
                               int* height, unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const long long base = claim_tickets(counter, 32);
    if (base >= nvert)
      break;
    const long long t = base + lane;
    if (t >= nvert)
      continue;
    const int u = nvert - 1 - (int)t;
    int h = 0;
    for (int p = __ldg(succptr + u); p < __ldg(succptr + u + 1); ++p) {
      const int w = __ldg(succ + p);
      const int hw = poll_nonneg_i32(height + w) + 1;
      h = hw > h ? hw : h;
    }
    st_relaxed_i32(height + u, h);
  }
}

__global__ void slack_kernel(const int32_t* __restrict__ level,
                             const int32_t* __restrict__ height, int32_t P,
                             int32_t nvert, int32_t* __restrict__ slack) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvert;
       v += (int64_t)gridDim.x * blockDim.x)
    slack[v] = P - level[v] - height[v];
}

__global__ void ascend_kernel(const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ idx, int32_t nvert,
                              int* bad) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nvert;
       u += (int64_t)gridDim.x * blockDim.x)
    for (int32_t p = ptr[u]; p < ptr[u + 1]; ++p)
      if (idx[p] <= u)
        *bad = 1;
}

__global__ void iota_kernel(int32_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void wave_ptr_kernel(const int32_t* __restrict__ sorted_levels,
                                int64_t n, int32_t P, int64_t* __restrict__ wp) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l <= P;
       l += (int64_t)gridDim.x * blockDim.x) {
    // wave l (1-based) starts at the first vertex with level >= l + 1 - 1
    const int32_t key = (int32_t)l + 1;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted_levels[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    wp[l] = lo;
  }
}

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 62 && (1ll << b) <= maxval)
    ++b;
  return b;
}

int grid_resident(const void* kernel) {
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
  return (per_sm < 1 ? 1 : per_sm) * sm_count();
}

} // namespace

void csr_from_edge_keys(DBuf<uint64_t>& keys, int64_t ne, int32_t nvert,
                        DevDag& out, cudaStream_t s) {
  out.nvert = nvert;
  out.ptr.alloc((int64_t)nvert + 1);
  int64_t nu = 0;
  DBuf<uint64_t> sorted;
  if (ne > 0) {
    TmpBuf<uint64_t> tmpk(ne, s);
    size_t bytes = 0;
    SFG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, tmpk.p, (int)ne, 0, 64, s));
    {
      TmpBuf<char> tmp((int64_t)bytes, s);
      SFG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, keys.p, tmpk.p, (int)ne, 0, 64, s));
    }
    TmpBuf<int64_t> nsel(1, s);
    bytes = 0;
    SFG_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, tmpk.p, keys.p, nsel.p, (int)ne, s));
    {
      TmpBuf<char> tmp((int64_t)bytes, s);
      SFG_CUDA(cub::DeviceSelect::Unique(tmp.p, bytes, tmpk.p, keys.p, nsel.p, (int)ne, s));
    }
    SFG_CUDA(cudaMemcpyAsync(&nu, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    // filtered entries carry the all-ones key and sort last
    if (nu > 0) {
      uint64_t last = 0;
      SFG_CUDA(cudaMemcpy(&last, keys.p + nu - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
      if (last == ~0ull)
        --nu;
    }
  }
  out.nedges = nu;
  out.idx.alloc(nu > 0 ? nu : 1);
  ptr_from_keys_kernel<<<grid_for(nu > nvert ? nu : (int64_t)nvert + 1), 256, 0, s>>>(
      keys.p, nu, nvert, out.ptr.p, out.idx.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void flip_dag(const DevDag& g, DevDag& out, cudaStream_t s) {
  DBuf<uint64_t> keys(g.nedges > 0 ? g.nedges : 1);
  if (g.nedges > 0) {
    flip_keys_kernel<<<grid_for((int64_t)g.nvert * 32), 256, 0, s>>>(g.ptr.p, g.idx.p,
                                                                     g.nvert, keys.p);
    count_launch();
  }
  csr_from_edge_keys(keys, g.nedges, g.nvert, out, s);
}

int32_t levels_syncfree(const int32_t* ptr, const int32_t* idx, int32_t nvert,
                        int dir, int32_t* level, cudaStream_t s) {
  if (nvert == 0)
    return 0;
  TmpBuf<unsigned long long> counter(1, s);
  SFG_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), s));
  SFG_CUDA(cudaMemsetAsync(level, 0, sizeof(int32_t) * (size_t)nvert, s));
  int64_t blocks = ((int64_t)nvert + 255) / 256;
  const int64_t cap = grid_resident((const void*)levels_kernel);
  if (blocks > cap)
    blocks = cap;
  levels_kernel<<<(unsigned)blocks, 256, 0, s>>>(ptr, idx, nvert, dir, level, counter.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  TmpBuf<int32_t> pmax(1, s);
  size_t bytes = 0;
  SFG_CUDA(cub::DeviceReduce::Max(nullptr, bytes, level, pmax.p, nvert, s));
  TmpBuf<char> tmp((int64_t)bytes, s);
  SFG_CUDA(cub::DeviceReduce::Max(tmp.p, bytes, level, pmax.p, nvert, s));
  int32_t P = 0;
  SFG_CUDA(cudaMemcpyAsync(&P, pmax.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  return P;
}

void heights_syncfree(const int32_t* succptr, const int32_t* succ,
                      int32_t nvert, int32_t* height, cudaStream_t s) {
  if (nvert == 0)
    return;
  TmpBuf<unsigned long long> counter(1, s);
  SFG_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), s));
  SFG_CUDA(cudaMemsetAsync(height, 0xFF, sizeof(int32_t) * (size_t)nvert, s));
  int64_t blocks = ((int64_t)nvert + 255) / 256;
  const int64_t cap = grid_resident((const void*)heights_kernel);
  if (blocks > cap)
    blocks = cap;
  heights_kernel<<<(unsigned)blocks, 256, 0, s>>>(succptr, succ, nvert, height, counter.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void slack_from(const int32_t* level, const int32_t* height, int32_t P,
                int32_t nvert, int32_t* slack, cudaStream_t s) {
  if (nvert == 0)
    return;
  slack_kernel<<<grid_for(nvert), 256, 0, s>>>(level, height, P, nvert, slack);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

bool edges_ascend(const DevDag& g, cudaStream_t s) {
  if (g.nvert == 0)
    return true;
  TmpBuf<int> bad(1, s);
  SFG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  ascend_kernel<<<grid_for(g.nvert), 256, 0, s>>>(g.ptr.p, g.idx.p, g.nvert, bad.p);
  count_launch();
  int h = 0;
  SFG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

void order_by_level(const int32_t* level, int32_t nvert, int32_t P,
                    int32_t* order, std::vector<int64_t>* wave_ptr,
                    cudaStream_t s) {
  if (nvert == 0) {
    if (wave_ptr)
      wave_ptr->assign(1, 0);
    return;
  }
  TmpBuf<int32_t> iota(nvert, s), sorted(nvert, s);
  iota_kernel<<<grid_for(nvert), 256, 0, s>>>(iota.p, nvert);
  count_launch();
  size_t bytes = 0;
  const int end_bit = bits_for(P);
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, level, sorted.p, iota.p, order,
                                           nvert, 0, end_bit, s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, level, sorted.p, iota.p, order,
                                             nvert, 0, end_bit, s));
  }
  if (wave_ptr) {
    TmpBuf<int64_t> wp((int64_t)P + 1, s);
    wave_ptr_kernel<<<grid_for((int64_t)P + 1), 256, 0, s>>>(sorted.p, nvert, P, wp.p);
    count_launch();
    wave_ptr->assign((size_t)P + 1, 0);
    SFG_CUDA(cudaMemcpyAsync(wave_ptr->data(), wp.p, sizeof(int64_t) * ((size_t)P + 1),
                             cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
  }
  SFG_CUDA(cudaGetLastError());
}

} // namespace sfg
