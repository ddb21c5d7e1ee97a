// internal.hpp -- host-side declarations shared by the libsfgpu translation
// units (storage transforms, inspector, executor, C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sfg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidMatrix : std::runtime_error {
  int32_t index;
  InvalidMatrix(const std::string& w, int32_t i) : std::runtime_error(w), index(i) {}
};
struct InvalidArgument : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// A factorization error detected while building a plan (scaling_vector's
// "zero diagonal", kernels.hpp:299-309, thrown by make_state for combo 3).
struct FactorizationFailure : std::runtime_error {
  int32_t kind, index;
  FactorizationFailure(const std::string& w, int32_t k, int32_t i)
      : std::runtime_error(w), kind(k), index(i) {}
};

void cuda_check(cudaError_t e, const char* what);
#define SFG_CUDA(x) ::sfg::cuda_check((x), #x)

// Plan-lifetime device buffer.
template <typename T> struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  DBuf() = default;
  explicit DBuf(int64_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(int64_t count) {
    release();
    n = count;
    // 64 bytes of tail slack: bulk copies round their source range out to
    // 16-byte boundaries (chaintma.cu)
    if (count > 0)
      SFG_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)count + 64));
  }
  void release() {
    if (p)
      cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  bool empty() const { return p == nullptr; }
};

// Launch accounting (bench "gpu_launches"): every kernel we launch bumps it.
extern thread_local int64_t* g_launch_counter;
inline void count_launch(int k = 1) {
  if (g_launch_counter)
    *g_launch_counter += k;
}

int sm_count();

// ---------------------------------------------------------------------------
// Storage transforms (storage.cu) -- the L0 conversions of make_state on GPU.
// ---------------------------------------------------------------------------

// Stable transpose of a compressed matrix: entries of major m (ptr over
// nmajor) become entries of minor-major storage, ascending major inside each
// new row.  perm[q] = source position of output entry q.
void transpose(const int32_t* ptr, const int32_t* idx, int32_t nmajor,
               int32_t nminor, int64_t nnz, int32_t* out_ptr, int32_t* out_idx,
               int32_t* perm, cudaStream_t s);

// Gather values for `nsys` systems: out[q*S + s] = in[s*in_stride + perm[q]]
// (in system-major, out interleaved).  perm == nullptr means identity.
void gather_values(const double* in, int64_t in_stride, const int32_t* perm,
                   int64_t nnz, int32_t nsys, double* out, cudaStream_t s);

// lower_triangle (matrix.hpp:98-128) of a CSC matrix: entries with row >= col.
// Returns the lower nnz; throws InvalidMatrix(column) on a missing or zero
// diagonal (checked for every system's values).  src_pos[q] = position in M.
int64_t lower_triangle(const int32_t* colptr, const int32_t* rowidx,
                       const double* vals, int64_t val_stride, int32_t nsys,
                       int32_t n, DBuf<int32_t>& lptr, DBuf<int32_t>& lidx,
                       DBuf<int32_t>& src_pos, cudaStream_t s);

// Reverse the entries of every compressed row/column (Lt = reversed CSC of L).
void reverse_segments(const int32_t* ptr, const int32_t* idx, int32_t nseg,
                      int32_t* out_idx, int32_t* perm, cudaStream_t s);

// diag position per CSR row (kernels.hpp:288-297); -1 if absent.
void find_diag_positions(const int32_t* rowptr, const int32_t* colidx,
                         int32_t n, int32_t* diag, cudaStream_t s);

// d[j] = 1 / sqrt(|L_jj|) with L_jj the first entry of CSC column j
// (kernels.hpp:485-487).
// scaling_vector (kernels.hpp:299-309) from CSR diagonal positions:
// d_i = 1 / sqrt(|a_ii|); returns the first row with a zero or missing
// diagonal, or -1.
int32_t scaling_vector_csr(const int32_t* diag, const double* vals, int32_t n, double* d,
                           cudaStream_t s);
void dscal_vector(const int32_t* colptr, const double* vals, int32_t n,
                  double* d, cudaStream_t s);

// Interleave / de-interleave nsys vectors of length n.
void interleave(const double* sys_major, int32_t n, int32_t nsys,
                double* inter, cudaStream_t s);
void deinterleave(const double* inter, int32_t n, int32_t nsys,
                  double* sys_major, cudaStream_t s);

// ---------------------------------------------------------------------------
// Inspector (inspector.cu)
// ---------------------------------------------------------------------------

// A DAG / dependence relation in CSR form on the device.
struct DevDag {
  int32_t nvert = 0;
  int64_t nedges = 0;
  DBuf<int32_t> ptr; // nvert+1
  DBuf<int32_t> idx; // nedges
  DBuf<int64_t> cost;
};

// Sort 64-bit (u<<32|v) edge keys, drop duplicates and build the CSR of the
// sources.  Consumes `keys` (length ne).
void csr_from_edge_keys(DBuf<uint64_t>& keys, int64_t ne, int32_t nvert,
                        DevDag& out, cudaStream_t s);

// Flip a CSR relation (succ -> pred), sorted.
void flip_dag(const DevDag& g, DevDag& out, cudaStream_t s);

// Sync-free longest-path levels over a predecessor structure: level[v] =
// 1 + max(level[u]); preds of v are idx[ptr[v]..ptr[v+1]) restricted to
// u < v (dir = +1, tickets ascending) or u > v (dir = -1, descending).
// Returns the critical path P.
int32_t levels_syncfree(const int32_t* ptr, const int32_t* idx, int32_t nvert,
                        int dir, int32_t* level, cudaStream_t s);
// Heights (longest path to a sink, in edges) over successor CSR, u < v edges.
void heights_syncfree(const int32_t* succptr, const int32_t* succ,
                      int32_t nvert, int32_t* height, cudaStream_t s);
void slack_from(const int32_t* level, const int32_t* height, int32_t P,
                int32_t nvert, int32_t* slack, cudaStream_t s);
// Checks every edge ascends (level_info's "edge does not ascend").
bool edges_ascend(const DevDag& g, cudaStream_t s);

// Stable order of vertices by level (the wavefront / ticket order).  Writes
// order[nvert] and (on the host) the wave boundaries.
void order_by_level(const int32_t* level, int32_t nvert, int32_t P,
                    int32_t* order, std::vector<int64_t>* wave_ptr,
                    cudaStream_t s);

} // namespace sfg
