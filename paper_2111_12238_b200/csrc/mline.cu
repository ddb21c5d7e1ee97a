// mline.cu -- inspector and executor of the multi-chain warp scheme (see
// mline.cuh).
#ifndef SFG_ML1_UNROLL
// unroll factor of k_mline1's step loop: with ring sizes that are powers of
// two, 8 turns every ring index into a compile-time constant (C1 kernel
// 0.589 -> 0.576 ms from the ring sizes, -> 0.535 ms at 8; 4: 0.576, 16: 0.599)
#define SFG_ML1_UNROLL 8
#endif
#include "common.cuh"
#include "mline.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <string>
#include <vector>

namespace sfg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kMThreads = 64; // 2 warps per CTA (several CTAs per SM as smem allows)

// Pipeline distances, in steps, for a lookahead DX: external x words are
// gathered DX steps ahead, values DV = DX+1, dependency codes DC = 2 DX and
// row pointers DP = 3 DX ahead, so every operand a stage reads was copied by
// a commit group at least DX iterations old (cp.async.wait_group DX-1).
template <int DX> struct Dist {
  static constexpr int DV = DX + 1, DC = 2 * DX, DP = 3 * DX;
  static constexpr int QX = DX + 1, QV = DV + 1, QC = DC + 1, QP = DP - DC + 1;
};

inline unsigned mgrid(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * 32;
  if (g > cap)
    g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

__device__ __forceinline__ int pos_of(int j, int n, int dir) { return dir > 0 ? j : n - 1 - j; }

// ---------------------------------------------------------------------------
// inspector
// ---------------------------------------------------------------------------

// One thread per group: skews of its chains in order (an earlier chain's
// skew is final before a later chain reads it) and the group's step count.
__global__ void group_skew_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  int32_t n, int dir, const int32_t* __restrict__ cstart,
                                  const int32_t* __restrict__ chain_of, int32_t nchain, int32_t B,
                                  int32_t ngroup, int32_t* cskew, int32_t* __restrict__ gsteps) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroup;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)g * B;
    const int nb = min(B, nchain - c0);
    const int gp0 = cstart[c0];
    int T = 0;
    for (int b = 0; b < nb; ++b) {
      const int c = c0 + b;
      const int p0 = cstart[c];
      const int len = cstart[c + 1] - p0;
      int sk = 0;
      for (int o = 0; o < len; ++o) {
        const int p = p0 + o;
        const int r = dir > 0 ? p : n - 1 - p;
        const int e1 = ptr[r + 1] - 1;
        for (int e = ptr[r]; e < e1; ++e) {
          const int pj = pos_of(idx[e], n, dir);
          if (pj >= gp0 && pj < p0) {
            const int cj = chain_of[pj];
            const int need = cskew[cj] + (pj - cstart[cj]) - o + 1;
            sk = need > sk ? need : sk;
          }
        }
      }
      cskew[c] = sk;
      T = sk + len > T ? sk + len : T;
    }
    gsteps[g] = T;
  }
}

// One thread per position: dependency codes (ring or external) and the
// group-DAG edge keys (group << 32 | dependency group; all-ones if internal).
__global__ void codes_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                             int32_t n, int dir, const int32_t* __restrict__ cstart,
                             const int32_t* __restrict__ chain_of, const int32_t* __restrict__ cskew,
                             int32_t B, int32_t* __restrict__ code, uint64_t* __restrict__ keys,
                             int* width) {
  int wmax = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int c = chain_of[p];
    const int g = c / B;
    const int c0 = g * B;
    const int gp0 = cstart[c0];
    const int o = (int)p - cstart[c];
    const int step = cskew[c] + o;
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int e0 = ptr[r], e1 = ptr[r + 1] - 1;
    const int nd = e1 - e0 - (o > 0 ? 1 : 0);
    wmax = nd > wmax ? nd : wmax;
    for (int e = e0; e < e1; ++e) {
      const int j = idx[e];
      const int pj = pos_of(j, n, dir);
      int cd = j;
      uint64_t key = ~0ull;
      if (pj >= gp0) {
        const int cj = chain_of[pj];
        const int delta = step - (cskew[cj] + (pj - cstart[cj]));
        if (delta >= 1 && delta < kRing)
          cd = -1 - (delta * 32 + (cj - c0));
      } else {
        const int gj = chain_of[pj] / B;
        key = ((uint64_t)(uint32_t)g << 32) | (uint32_t)gj;
      }
      code[e] = cd;
      keys[e] = key;
    }
    code[e1] = r;
    keys[e1] = ~0ull;
  }
  atomicMax(width, wmax);
}


// One warp per group, claimed in group-DAG level order.  est[g] is the
// group's earliest start in 1/64 steps given its predecessors' (real lags,
// which are negative where a producer row comes later in its group than the
// consumer row in this one); key[g] = max(est[g], key[h] + 1 over
// predecessors) is the claim priority -- est order made topological, so
// skewed neighbours are claimed together instead of being serialised.
// key_p1 holds key + 1 (0 = not final yet); every predecessor was claimed
// earlier.
__global__ void group_est_kernel(const int32_t* __restrict__ ptr, int32_t n, int dir,
                                 const int32_t* __restrict__ cstart,
                                 const int32_t* __restrict__ chain_of,
                                 const int32_t* __restrict__ cskew,
                                 const int32_t* __restrict__ code,
                                 const int32_t* __restrict__ gorder, int32_t ng, int32_t nchain,
                                 int32_t B, int hop, int32_t* est, int32_t* key_p1,
                                 unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0)
      t = atomicAdd(counter, 1ull);
    t = __shfl_sync(FULL, t, 0);
    if (t >= (unsigned long long)ng)
      break;
    const int g = gorder[t];
    int best = 0, kbest = 0;
    for (int b = lane; b < B; b += 32) {
      const int c = g * B + b;
      if (c >= nchain)
        break;
      const int p0 = cstart[c], len = cstart[c + 1] - p0, sk = cskew[c];
      for (int o = 0; o < len; ++o) {
        const int p = p0 + o;
        const int r = dir > 0 ? p : n - 1 - p;
        for (int e = ptr[r]; e < ptr[r + 1] - 1; ++e) {
          const int cd = code[e];
          if (cd < 0)
            continue;
          const int pj = pos_of(cd, n, dir);
          const int cj = chain_of[pj];
          const int h = cj / B;
          if (h == g)
            continue;
          int kv;
          while ((kv = *(volatile int32_t*)(key_p1 + h)) == 0)
            ;
          const int ev = *(volatile int32_t*)(est + h);
          const int w = (cskew[cj] + (pj - cstart[cj]) - (sk + o) + 1 + hop) * 64;
          best = ev + w > best ? ev + w : best;
          kbest = kv > kbest ? kv : kbest; // key[h] + 1
        }
      }
    }
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      const int v = __shfl_xor_sync(FULL, best, o2);
      best = v > best ? v : best;
      const int kk = __shfl_xor_sync(FULL, kbest, o2);
      kbest = kk > kbest ? kk : kbest;
    }
    if (lane == 0) {
      *(volatile int32_t*)(est + g) = best;
      __threadfence();
      *(volatile int32_t*)(key_p1 + g) = (best > kbest ? best : kbest) + 1;
      __threadfence();
    }
    __syncwarp();
  }
}

// One thread per position: its step-stream record (S == 1).
__global__ void stream_fill_kernel(const int32_t* __restrict__ ptr, const double* __restrict__ val,
                                   int32_t n, int dir, const int32_t* __restrict__ cstart,
                                   const int32_t* __restrict__ chain_of,
                                   const int32_t* __restrict__ cskew,
                                   const int32_t* __restrict__ code,
                                   const int64_t* __restrict__ sofs, int32_t* __restrict__ srow,
                                   int32_t* __restrict__ scode, double* __restrict__ sval,
                                   int ch, int* too_wide) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int c = chain_of[p];
    const int g = c >> 5, b = c & 31;
    const int o = (int)p - cstart[c];
    const int64_t rec = sofs[g] + (int64_t)(cskew[c] + o) * 32 + b;
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int e0 = ptr[r], e1 = ptr[r + 1];
    const bool chained = o > 0;
    const int nd = e1 - e0 - 1 - (chained ? 1 : 0);
    if (nd > ch) {
      atomicOr(too_wide, 1);
      continue;
    }
    srow[rec] = r;
    for (int a = 0; a < ch; ++a) {
      scode[rec * ch + a] = a < nd ? code[e0 + a] : n; // padding: the zero row
      sval[rec * (ch + 4) + a] = a < nd ? val[e0 + a] : 0.0;
    }
    sval[rec * (ch + 4) + ch] = chained ? val[e1 - 2] : 0.0;
    sval[rec * (ch + 4) + ch + 1] = val[e1 - 1];
    sval[rec * (ch + 4) + ch + 2] = __drcp_rn(val[e1 - 1]); // reciprocal off the step's chain
    sval[rec * (ch + 4) + ch + 3] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// executor
// ---------------------------------------------------------------------------

template <int S, int CHN, int DX> struct MlWarp {
  static constexpr int B = 32 / S;
  using D = Dist<DX>;
  int32_t code[D::QC][B][CHN];
  int32_t meta[D::QC][B][4]; // row (-1 = idle), first dependency entry, #deps, chained
  int32_t rptr[D::QP][B][2];
  double v[D::QV][B][CHN + 2][S]; // deps, carry coefficient, diagonal
  unsigned long long x[D::QX][B][CHN][S];
  unsigned long long rhs[D::QV][B][S];
  double ring[kRing][32];
};

__device__ __forceinline__ void cp8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  // no "memory" clobber: the copy's destination is only read after a
  // cp.async.wait_group (which has one), so the compiler may interleave the
  // stages' independent shared-memory loads with the copy issue
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int S, int CHN, int DX>
__global__ void __launch_bounds__(kMThreads) k_mline(const MLineArgs A) {
  constexpr int B = 32 / S;
  using D = Dist<DX>;
  constexpr int DV = D::DV, DC = D::DC, DP = D::DP;
  constexpr int QX = D::QX, QV = D::QV, QC = D::QC, QP = D::QP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MlWarp<S, CHN, DX>& W = reinterpret_cast<MlWarp<S, CHN, DX>*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int b = lane / S;
  const int s = lane % S;
  const int total = A.seg_end - A.seg_begin;
  for (;;) {
    unsigned long long w0 = 0;
    if (lane == 0)
      w0 = atomicAdd(A.counter, 1ull);
    const long long wi = (long long)__shfl_sync(FULL, w0, 0);
    if (wi >= total)
      break;
    const int item = A.seg_begin + (int)wi;
    const bool spmv4 = A.combo == 4 && item >= A.f_ngroup;
    const bool spmv2 = A.combo == 2 && item < A.f_ngroup;
    if (S == 1 && (spmv4 || spmv2)) {
      // SpMV rows blk * 32 + lane as a row gather over CSR(A) in ascending
      // column order.  Combo 4 kernel 2: the order in which the sequential
      // CSC scatter (spmv_csc_col, kernels.hpp:162-168) accumulates y_r,
      // over the solved vector; combo 2 kernel 1: spmv_csr_row
      // (kernels.hpp:152-158) over the input vector, published for the solve.
      const int blk = spmv4 ? item - A.f_ngroup : item;
      const double* xsrc = spmv4 ? A.vmid : A.vin;
      const int r = blk * 32 + lane;
      if (spmv4) {
        // one lane watches the block's newest operand (the last row's
        // largest column) with a long back-off before the block gathers
        const int rl = min(blk * 32 + 31, A.n - 1);
        if (lane == 0) {
          const int pl = __ldg(A.ar_ptr + rl + 1) - 1;
          if (pl >= 0) {
            const int jl = __ldg(A.ar_idx + pl);
            while (is_sent_hi(ld_relaxed_u64(A.vmid + jl)))
              __nanosleep(1000);
          }
        }
        __syncwarp();
      }
      if (r < A.n) {
        const int pb = __ldg(A.ar_ptr + r), pe = __ldg(A.ar_ptr + r + 1);
        double acc = 0.0;
        for (int p = pb; p < pe; p += 8) {
          const int cnt = pe - p < 8 ? pe - p : 8;
          int jj[8];
          unsigned long long ww[8];
#pragma unroll
          for (int a = 0; a < 8; ++a)
            if (a < cnt)
              jj[a] = __ldg(A.ar_idx + p + a);
          // wait for the whole batch with a long back-off: these warps have
          // nothing else to do and must not steal L2 bandwidth or issue
          // slots from the solve they wait on
          for (bool first = true;; first = false) {
            bool pending = false;
#pragma unroll
            for (int a = 0; a < 8; ++a)
              if (a < cnt && (first || is_sent_hi(ww[a]))) {
                ww[a] = ld_relaxed_u64(xsrc + jj[a]);
              }
#pragma unroll
            for (int a = 0; a < 8; ++a)
              pending |= a < cnt && is_sent_hi(ww[a]);
            if (!pending)
              break;
            __nanosleep(1000);
          }
#pragma unroll
          for (int a = 0; a < 8; ++a)
            if (a < cnt)
              acc = __dadd_rn(acc, __dmul_rn(__ldg(A.ar_val + p + a),
                                             __longlong_as_double((long long)ww[a])));
        }
        if (spmv4)
          A.vout[r] = acc;
        else
          publish_f64(A.vmid + r, acc);
      }
      continue;
    }
    const bool second = item >= A.f_ngroup;
    const bool bwd = second && A.combo == 8;
    const int32_t* ptr = bwd ? A.lt_ptr : A.lr_ptr;
    const double* val = bwd ? A.lt_val : A.lr_val;
    const int32_t* code = bwd ? A.b_code : A.f_code;
    const int32_t* cstart = bwd ? A.b_cstart : A.f_cstart;
    const int32_t* cskew = bwd ? A.b_cskew : A.f_cskew;
    const int nchain = bwd ? A.b_nchain : A.f_nchain;
    const int g = second ? __ldg((bwd ? A.b_gorder : A.f_gorder) + (item - A.f_ngroup))
                         : __ldg(A.f_gorder + item);
    const int T = __ldg((bwd ? A.b_gsteps : A.f_gsteps) + g);
    const int c = g * B + b;
    const bool has_chain = c < nchain;
    const int p0 = has_chain ? __ldg(cstart + c) : 0;
    const int len = has_chain ? __ldg(cstart + c + 1) - p0 : 0;
    const int skew = has_chain ? __ldg(cskew + c) : 0;
    double* xo = second ? A.vout : A.vmid;
    const double* rhs_vec = second ? A.vmid : A.vin;
    const int kern = second ? 2 : 1;
    auto row_of = [&](int o) {
      const int p = p0 + o;
      return bwd ? A.n - 1 - p : p;
    };
    double carry = 0.0;
    unsigned long long tr_claim = 0, tr_first = 0, wait_cyc = 0, poll_cyc = 0;
    if (A.trace)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_claim));
    __syncwarp();
    // Every global operand reaches shared memory through cp.async, one
    // commit group per iteration, so no load result is carried across
    // iterations in a register (a register hand-off would stall the warp on
    // the load at the end of every step).
#pragma unroll 1
    for (int i = -DP; i < T; ++i) {
      if (A.trace && i == 0)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_first));
      // commit groups <= i-DX complete: row pointers of step i+DC, codes of
      // step i+DX, values and gathered x of step i
      const long long wc0 = A.trace ? clock64() : 0;
      cp_wait<DX - 1>();
      __syncwarp();
      if (A.trace)
        wait_cyc += clock64() - wc0;
      // ---- stage A: row pointers of step i+DP
      if (i + DP >= 0) {
        const int o = i + DP - skew;
        if (s == 0 && o >= 0 && o < len) {
          const int r = row_of(o);
          cp4(&W.rptr[(i + DP) % QP][b][0], ptr + r);
          cp4(&W.rptr[(i + DP) % QP][b][1], ptr + r + 1);
        }
      }
      // ---- stage B': meta + dependency codes of step i+DC
      if (i + DC >= 0) {
        const int q = (i + DC) % QC;
        const int o = i + DC - skew;
        const bool act = o >= 0 && o < len;
        const bool chained = o > 0;
        const int r = act ? row_of(o) : -1;
        const int e0 = act ? W.rptr[(i + DC) % QP][b][0] : 0;
        const int e1 = act ? W.rptr[(i + DC) % QP][b][1] : 0;
        const int nd = act ? e1 - e0 - 1 - (chained ? 1 : 0) : 0;
        if (s == 0) {
          W.meta[q][b][0] = r;
          W.meta[q][b][1] = e0;
          W.meta[q][b][2] = nd;
          W.meta[q][b][3] = chained ? 1 : 0;
        }
        if (act) {
          const int m = nd < CHN ? nd : CHN;
          for (int a = s; a < m; a += S)
            cp4(&W.code[q][b][a], code + e0 + a);
        }
      }
      __syncwarp();
      // ---- stage B: values and right-hand side of step i+DV
      if (i + DV >= 0) {
        const int q = (i + DV) % QC;
        const int qv = (i + DV) % QV;
        const int r = W.meta[q][b][0];
        if (r >= 0) {
          const int e0 = W.meta[q][b][1];
          const int nd = W.meta[q][b][2];
          const bool chained = W.meta[q][b][3] != 0;
          const int m = nd < CHN ? nd : CHN;
          const double* vb = val + (size_t)e0 * S + s;
#pragma unroll
          for (int a = 0; a < CHN; ++a)
            if (a < m)
              cp8(&W.v[qv][b][a][s], vb + (size_t)a * S);
          const int ediag = e0 + nd + (chained ? 1 : 0);
          if (chained)
            cp8(&W.v[qv][b][CHN][s], val + (size_t)(ediag - 1) * S + s);
          cp8(&W.v[qv][b][CHN + 1][s], val + (size_t)ediag * S + s);
          cp8(&W.rhs[qv][b][s], rhs_vec + (size_t)r * S + s);
        }
      }
      // ---- stage C: gather the external x words of step i+DX
      if (i + DX >= 0) {
        const int q = (i + DX) % QC;
        const int qx = (i + DX) % QX;
        if (W.meta[q][b][0] >= 0) {
          const int nd = W.meta[q][b][2];
          const int m = nd < CHN ? nd : CHN;
#pragma unroll
          for (int a = 0; a < CHN; ++a)
            if (a < m) {
              const int cd = W.code[q][b][a];
              if (cd >= 0)
                cp8(&W.x[qx][b][a][s], xo + (size_t)cd * S + s);
            }
        }
      }
      cp_commit();
      // ---- stage D: row of step i
      if (i >= 0) {
        const int q = i % QC;
        const int qv = i % QV;
        const int qx = i % QX;
        const int r = W.meta[q][b][0];
        if (r >= 0) {
          const int e0 = W.meta[q][b][1];
          const int nd = W.meta[q][b][2];
          const bool chained = W.meta[q][b][3] != 0;
          const int m = nd < CHN ? nd : CHN;
          const double d = W.v[qv][b][CHN + 1][s];
          const double rd = __drcp_rn(d);
          unsigned long long rw = W.rhs[qv][b][s];
          int cds[CHN];
          unsigned long long wd[CHN];
#pragma unroll
          for (int a = 0; a < CHN; ++a)
            if (a < m) {
              const int cd = W.code[q][b][a];
              cds[a] = cd;
              if (cd >= 0) {
                wd[a] = W.x[qx][b][a][s];
              } else {
                const int t = -1 - cd;
                wd[a] = (unsigned long long)__double_as_longlong(
                    W.ring[(i - (t >> 5)) & (kRing - 1)][(t & 31) * S + s]);
              }
            }
          // re-poll words that were still unpublished when gathered
          const long long pc0 = A.trace ? clock64() : 0;
          for (;;) {
            bool pending = is_sent_hi(rw);
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              pending |= a < m && is_sent_hi(wd[a]);
            if (!pending)
              break;
            if (A.sleep_ns)
              __nanosleep(A.sleep_ns);
            if (is_sent_hi(rw))
              rw = ld_relaxed_u64(rhs_vec + (size_t)r * S + s);
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < m && is_sent_hi(wd[a]))
                wd[a] = ld_relaxed_u64(xo + (size_t)cds[a] * S + s);
          }
          if (A.trace)
            poll_cyc += clock64() - pc0;
          double acc = __longlong_as_double((long long)rw);
#pragma unroll
          for (int a = 0; a < CHN; ++a)
            if (a < m)
              acc = __dsub_rn(acc, __dmul_rn(W.v[qv][b][a][s], __longlong_as_double((long long)wd[a])));
          for (int e = e0 + CHN; e < e0 + nd; ++e) { // rows wider than the staging
            const int cd = __ldg(code + e);
            double xv;
            if (cd >= 0) {
              xv = poll_f64(xo + (size_t)cd * S + s, 0);
            } else {
              const int t = -1 - cd;
              xv = W.ring[(i - (t >> 5)) & (kRing - 1)][(t & 31) * S + s];
            }
            acc = __dsub_rn(acc, __dmul_rn(__ldg(val + (size_t)e * S + s), xv));
          }
          if (chained)
            acc = __dsub_rn(acc, __dmul_rn(W.v[qv][b][CHN][s], carry));
          if (d == 0.0)
            report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
          const double xv = div_with_rcp(acc, d, rd);
          publish_f64(xo + (size_t)r * S + s, xv);
          W.ring[i & (kRing - 1)][lane] = xv;
          carry = xv;
        }
      }
      __syncwarp();
    }
    cp_wait0();
    __syncwarp();
    if (A.trace) {
      unsigned long long pmax = poll_cyc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(FULL, pmax, o);
        pmax = v > pmax ? v : pmax;
      }
      if (lane == 0) {
        unsigned long long te;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        unsigned long long* tr = A.trace + (size_t)item * 4;
        tr[0] = tr_claim;
        tr[1] = tr_first;
        tr[2] = te;
        tr[3] = (wait_cyc << 32) | (pmax & 0xffffffffull);
      }
    }
  }
}

// Single-system multi-chain executor on the step stream: lane b owns chain
// b of the group; per step it copies its own record (4 dependency codes, 6
// values, row) with coalesced 16-byte copies kRA1 steps ahead, gathers the
// right-hand side and the external dependency words kXA1 steps ahead, and
// completes its row from shared memory (ring for in-group dependencies).
constexpr int kXA1 = 2;        // gathers run kXA1 steps ahead
constexpr int kRA1 = 2 * kXA1; // records run kRA1 steps ahead
constexpr int kQ1 = 8;         // record slots (a power of two >= kRA1 + 1): steps i .. i+kRA1
constexpr int kX1 = 4;         // gathered-word slots (a power of two >= kXA1 + 1): steps i .. i+kXA1
static_assert(kQ1 >= kRA1 + 1 && kX1 >= kXA1 + 1 && (kQ1 & (kQ1 - 1)) == 0 && (kX1 & (kX1 - 1)) == 0, "ring sizes");
template <int CH> struct alignas(16) Ml1Warp {
  double v[kQ1][32][CH + 4]; // deps, carry coefficient, diagonal, its reciprocal, pad
  int32_t cd[kQ1][32][CH];
  int32_t row[kQ1][32];
  unsigned long long x[kX1][32][CH];
  unsigned long long rhs[kX1][32];
  double ring[kRing][32];
};

#ifndef SFG_ML1_TRACE
#define SFG_ML1_TRACE 0 // 1: k_mline1 records its timeline when SFG_TRACE is set (diagnostic builds)
#endif
template <int CH>
__global__ void __launch_bounds__(kMThreads) k_mline1(const MLineArgs A) {
  static_assert(CH == 2 || CH == 4, "record widths of 32 or 48 bytes");
  const bool tracing = SFG_ML1_TRACE && A.trace;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ml1Warp<CH>& W = reinterpret_cast<Ml1Warp<CH>*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int total = A.seg_end - A.seg_begin;
  for (;;) {
    unsigned long long w0 = 0;
    if (lane == 0)
      w0 = atomicAdd(A.counter, 1ull);
    const long long wi = (long long)__shfl_sync(FULL, w0, 0);
    if (wi >= total)
      break;
    const int item = A.seg_begin + (int)wi;
    const bool spmv4 = A.combo == 4 && item >= A.f_ngroup;
    const bool spmv2 = A.combo == 2 && item < A.f_ngroup;
    if (spmv4 || spmv2) { // SpMV row blocks (see k_mline)
      const int blk = spmv4 ? item - A.f_ngroup : item;
      const double* xsrc = spmv4 ? A.vmid : A.vin;
      const int r = blk * 32 + lane;
      if (spmv4) {
        const int rl = min(blk * 32 + 31, A.n - 1);
        if (lane == 0) {
          const int pl = __ldg(A.ar_ptr + rl + 1) - 1;
          if (pl >= 0) {
            const int jl = __ldg(A.ar_idx + pl);
            while (is_sent_hi(ld_relaxed_u64(A.vmid + jl)))
              __nanosleep(1000);
          }
        }
        __syncwarp();
      }
      if (r < A.n) {
        double acc = 0.0;
        for (int p = __ldg(A.ar_ptr + r); p < __ldg(A.ar_ptr + r + 1); ++p) {
          const int j = __ldg(A.ar_idx + p);
          unsigned long long w = ld_relaxed_u64(xsrc + j);
          while (is_sent_hi(w)) {
            __nanosleep(1000);
            w = ld_relaxed_u64(xsrc + j);
          }
          acc = __dadd_rn(acc, __dmul_rn(__ldg(A.ar_val + p), __longlong_as_double((long long)w)));
        }
        if (spmv4)
          A.vout[r] = acc;
        else
          publish_f64(A.vmid + r, acc);
      }
      continue;
    }
    const bool second = item >= A.f_ngroup;
    const bool bwd = second && A.combo == 8;
    const int g = second ? __ldg((bwd ? A.b_gorder : A.f_gorder) + (item - A.f_ngroup))
                         : __ldg(A.f_gorder + item);
    const int T = __ldg((bwd ? A.b_gsteps : A.f_gsteps) + g);
    const int64_t base = __ldg((bwd ? A.b_sofs : A.f_sofs) + g) + lane;
    const int32_t* srow = bwd ? A.b_srow : A.f_srow;
    const int32_t* scode = bwd ? A.b_scode : A.f_scode;
    const double* sval = bwd ? A.b_sval : A.f_sval;
    double* xo = second ? A.vout : A.vmid;
    const double* rhs_vec = second ? A.vmid : A.vin;
    const int kern = second ? 2 : 1;
    double carry = 0.0;
    bool started = false;
    unsigned long long tr_claim = 0, tr_first = 0, poll_cyc = 0, d_cyc = 0;
    if (tracing)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_claim));
    __syncwarp();
#if SFG_ML1_UNROLL
    constexpr int kUnrollM = SFG_ML1_UNROLL;
#pragma unroll kUnrollM
#else
#pragma unroll 1
#endif
    for (int i = -kRA1; i < T; ++i) {
      if (tracing && i == 0)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_first));
      // commit groups <= i - kXA1 complete: records of steps <= i + kXA1,
      // gathers of steps <= i
      asm volatile("cp.async.wait_group %0;" ::"n"(kXA1 - 1) : "memory");
      __syncwarp();
      // ---- record of step i+kRA1
      if (i + kRA1 < T) {
        const int q = (i + kRA1) & (kQ1 - 1);
        const int64_t rec = base + (int64_t)(i + kRA1) * 32;
        const double* vr = sval + rec * (CH + 4);
#pragma unroll
        for (int h = 0; h < CH + 4; h += 2)
          cp16(&W.v[q][lane][h], vr + h);
        if (CH == 4)
          cp16(&W.cd[q][lane][0], scode + rec * CH);
        else
          cp8(&W.cd[q][lane][0], scode + rec * CH);
        cp4(&W.row[q][lane], srow + rec);
      }
      // ---- right-hand side and external words of step i+kXA1
      if (i + kXA1 >= 0 && i + kXA1 < T) {
        const int q = (i + kXA1) & (kQ1 - 1), qx = (i + kXA1) & (kX1 - 1);
        const int r = W.row[q][lane];
        if (r >= 0) {
          cp8(&W.rhs[qx][lane], rhs_vec + r);
#pragma unroll
          for (int a = 0; a < CH; ++a) {
            const int cd = W.cd[q][lane][a];
            if (cd >= 0)
              cp8(&W.x[qx][lane][a], xo + cd);
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      // ---- row of step i
      const long long dc0 = tracing ? clock64() : 0;
      if (i >= 0) {
        const int q = i & (kQ1 - 1), qx = i & (kX1 - 1);
        const int r = W.row[q][lane];
        if (r >= 0) {
          const double d = W.v[q][lane][CH + 1];
          const double rd = W.v[q][lane][CH + 2];
          unsigned long long rw = W.rhs[qx][lane];
          int cds[CH];
          unsigned long long wd[CH];
#pragma unroll
          for (int a = 0; a < CH; ++a) {
            const int cd = W.cd[q][lane][a];
            cds[a] = cd;
            if (cd >= 0) {
              wd[a] = W.x[qx][lane][a];
            } else {
              const int t = -1 - cd;
              wd[a] = (unsigned long long)__double_as_longlong(
                  W.ring[(i - (t >> 5)) & (kRing - 1)][t & 31]);
            }
          }
          const long long pc0 = tracing ? clock64() : 0;
          for (;;) {
            bool pending = is_sent_hi(rw);
#pragma unroll
            for (int a = 0; a < CH; ++a)
              pending |= is_sent_hi(wd[a]);
            if (!pending)
              break;
            if (is_sent_hi(rw))
              rw = ld_relaxed_u64(rhs_vec + r);
#pragma unroll
            for (int a = 0; a < CH; ++a)
              if (is_sent_hi(wd[a]))
                wd[a] = ld_relaxed_u64(xo + cds[a]);
          }
          if (tracing)
            poll_cyc += clock64() - pc0;
          double acc = __longlong_as_double((long long)rw);
#pragma unroll
          for (int a = 0; a < CH; ++a)
            acc = __dsub_rn(acc, __dmul_rn(W.v[q][lane][a], __longlong_as_double((long long)wd[a])));
          if (started)
            acc = __dsub_rn(acc, __dmul_rn(W.v[q][lane][CH], carry));
          if (d == 0.0)
            report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
          const double xv = div_with_rcp(acc, d, rd);
          publish_f64(xo + r, xv);
          W.ring[i & (kRing - 1)][lane] = xv;
          carry = xv;
          started = true;
        }
      }
      __syncwarp();
      if (tracing)
        d_cyc += clock64() - dc0;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (tracing) {
      unsigned long long pm = poll_cyc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(FULL, pm, o);
        pm = v > pm ? v : pm;
      }
      if (lane == 0) {
        unsigned long long te;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        unsigned long long* tr = A.trace + (size_t)item * 4;
        tr[0] = tr_claim;
        tr[1] = tr_first;
        tr[2] = te;
        tr[3] = (d_cyc << 32) | (pm & 0xffffffffull);
      }
    }
  }
}


template <int S, int CHN, int DX> void launch_scd(const MLineArgs& a, cudaStream_t s) {
  // single-system plans are latency-bound: one CTA per SM keeps the solve
  // warps from sharing schedulers with waiting warps (measured on C1)
  auto kern = k_mline<S, CHN, DX>;
  const size_t smem = (size_t)(kMThreads / 32) * sizeof(MlWarp<S, CHN, DX>);
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMThreads, smem));
  if (per_sm < 1)
    per_sm = 1;
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  else if (a.blocks_per_sm == 0 && S == 1)
    per_sm = 1;
  const int64_t items = a.seg_end - a.seg_begin;
  int64_t grid = (items + (kMThreads / 32) - 1) / (kMThreads / 32);
  if (grid > (int64_t)per_sm * sm_count())
    grid = (int64_t)per_sm * sm_count();
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, kMThreads, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

template <int S, int CHN> void launch_sc(const MLineArgs& a, cudaStream_t s) {
  if (a.lookahead <= 2)
    launch_scd<S, CHN, 2>(a, s);
  else
    launch_scd<S, CHN, 4>(a, s);
}

template <int S> void launch_s(const MLineArgs& a, cudaStream_t s) {
  if (a.chn <= 4)
    launch_sc<S, 4>(a, s);
  else
    launch_sc<S, 12>(a, s);
}

} // namespace

void build_mline(const int32_t* ptr, const int32_t* idx, int32_t n, int dir, int32_t S,
                 int32_t max_len, MLineLayout& out, cudaStream_t s) {
  out.n = n;
  out.S = S;
  out.B = 32 / S;
  out.dir = dir;
  const int32_t B = out.B;
  if (n == 0) {
    out.nchain = out.ngroup = out.nlevels = 0;
    out.cstart.alloc(1);
    SFG_CUDA(cudaMemsetAsync(out.cstart.p, 0, sizeof(int32_t), s));
    return;
  }
  // chains: maximal runs whose last dependency is the previous position
  ChainLayout ch;
  build_chains(ptr, idx, n, dir, 1, 1, max_len, ch, s);
  out.nchain = ch.nchain;
  out.cstart = std::move(ch.cstart);
  out.chain_of = std::move(ch.chain_of);
  const int32_t nc = out.nchain;
  out.ngroup = (nc + B - 1) / B;
  const int32_t ng = out.ngroup;
  out.cskew.alloc(nc);
  out.gsteps.alloc(ng);
  SFG_CUDA(cudaMemsetAsync(out.cskew.p, 0, sizeof(int32_t) * (size_t)nc, s));
  group_skew_kernel<<<mgrid(ng, 64), 64, 0, s>>>(ptr, idx, n, dir, out.cstart.p, out.chain_of.p, nc,
                                                  B, ng, out.cskew.p, out.gsteps.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  int32_t nnz = 0;
  SFG_CUDA(cudaMemcpyAsync(&nnz, ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  out.code.alloc(nnz > 0 ? nnz : 1);
  DBuf<uint64_t> keys(nnz > 0 ? nnz : 1);
  DBuf<int> width(1);
  SFG_CUDA(cudaMemsetAsync(width.p, 0, sizeof(int), s));
  codes_kernel<<<mgrid(n), 256, 0, s>>>(ptr, idx, n, dir, out.cstart.p, out.chain_of.p,
                                         out.cskew.p, B, out.code.p, keys.p, width.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaMemcpyAsync(&out.CHN, width.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  // group DAG -> levels -> claim order
  DevDag gd;
  csr_from_edge_keys(keys, nnz, ng, gd, s);
  DBuf<int32_t> level(ng);
  out.nlevels = levels_syncfree(gd.ptr.p, gd.idx.p, ng, +1, level.p, s);
  out.gorder.alloc(ng);
  order_by_level(level.p, ng, out.nlevels, out.gorder.p, nullptr, s);
  SFG_CUDA(cudaStreamSynchronize(s));
  out.glevel = std::move(level);
  // SFG_GROUP_ORDER=est: claim by earliest start instead of level (an
  // ablation; measured neutral on C5 with either multi-line executor)
  const char* go_env = getenv("SFG_GROUP_ORDER");
  const bool by_est = go_env && std::string(go_env) == "est";
  if (by_est && ng > 1) {
    DBuf<int32_t> est(ng), key(ng);
    SFG_CUDA(cudaMemsetAsync(est.p, 0, sizeof(int32_t) * (size_t)ng, s));
    SFG_CUDA(cudaMemsetAsync(key.p, 0, sizeof(int32_t) * (size_t)ng, s));
    DBuf<unsigned long long> ctr(1);
    SFG_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned long long), s));
    int hop = 2;
    if (const char* e = getenv("SFG_GROUP_HOP"))
      hop = atoi(e);
    int per_sm = 0;
    SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, group_est_kernel, 128, 0));
    const int64_t grid = std::min<int64_t>(((int64_t)ng + 3) / 4, (int64_t)std::max(per_sm, 1) * sm_count());
    group_est_kernel<<<(unsigned)grid, 128, 0, s>>>(ptr, n, dir, out.cstart.p, out.chain_of.p,
                                                   out.cskew.p, out.code.p, out.gorder.p, ng,
                                                   out.nchain, B, hop, est.p, key.p, ctr.p);
    count_launch();
    SFG_CUDA(cudaGetLastError());
    std::vector<int32_t> hk((size_t)ng), he((size_t)ng);
    SFG_CUDA(cudaMemcpyAsync(hk.data(), key.p, sizeof(int32_t) * (size_t)ng, cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaMemcpyAsync(he.data(), est.p, sizeof(int32_t) * (size_t)ng, cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    int32_t kmax = 0, emax = 0;
    for (size_t g = 0; g < hk.size(); ++g) {
      kmax = std::max(kmax, hk[g]);
      emax = std::max(emax, he[g]);
    }
    order_by_level(key.p, ng, kmax + 1, out.gorder.p, nullptr, s);
    SFG_CUDA(cudaStreamSynchronize(s));
    out.est_steps = emax / 64;
  }
  // longest group (diagnostics)
  std::vector<int32_t> hs((size_t)ng);
  SFG_CUDA(cudaMemcpyAsync(hs.data(), out.gsteps.p, sizeof(int32_t) * (size_t)ng,
                           cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  out.max_steps = 0;
  for (int32_t v : hs)
    out.max_steps = v > out.max_steps ? v : out.max_steps;
}

void build_mline_stream(const int32_t* ptr, const double* val, int32_t n, int dir,
                        MLineLayout& L, cudaStream_t s) {
  L.stream = false;
  if (L.S != 1 || L.ngroup == 0)
    return;
  std::vector<int32_t> gs((size_t)L.ngroup);
  SFG_CUDA(cudaMemcpyAsync(gs.data(), L.gsteps.p, sizeof(int32_t) * gs.size(),
                           cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> so((size_t)L.ngroup + 1, 0);
  for (int32_t g = 0; g < L.ngroup; ++g)
    so[(size_t)g + 1] = so[(size_t)g] + (int64_t)gs[(size_t)g] * 32;
  L.nrec = so[(size_t)L.ngroup];
  L.sofs.alloc((int64_t)L.ngroup + 1);
  SFG_CUDA(cudaMemcpyAsync(L.sofs.p, so.data(), sizeof(int64_t) * so.size(),
                           cudaMemcpyHostToDevice, s));
  L.sch = L.CHN <= 2 ? 2 : kStreamChn;
  L.srow.alloc(L.nrec > 0 ? L.nrec : 1);
  L.scode.alloc((L.nrec > 0 ? L.nrec : 1) * L.sch);
  L.sval.alloc((L.nrec > 0 ? L.nrec : 1) * (L.sch + 4));
  SFG_CUDA(cudaMemsetAsync(L.srow.p, 0xFF, sizeof(int32_t) * (size_t)std::max<int64_t>(L.nrec, 1), s));
  DBuf<int> wide(1);
  SFG_CUDA(cudaMemsetAsync(wide.p, 0, sizeof(int), s));
  stream_fill_kernel<<<mgrid(n), 256, 0, s>>>(ptr, val, n, dir, L.cstart.p, L.chain_of.p, L.cskew.p,
                                               L.code.p, L.sofs.p, L.srow.p, L.scode.p, L.sval.p,
                                               L.sch, wide.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  int hw = 0;
  SFG_CUDA(cudaMemcpyAsync(&hw, wide.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  L.stream = hw == 0;
  if (!L.stream) {
    L.srow.release();
    L.scode.release();
    L.sval.release();
  }
}

void launch_mline(const MLineArgs& a, cudaStream_t s) {
  if (a.seg_end <= a.seg_begin)
    return;
  if (a.S == 1 && a.use_stream) {
    auto kern = a.stream_ch <= 2 ? k_mline1<2> : k_mline1<4>;
    const size_t smem = (size_t)(kMThreads / 32) *
                        (a.stream_ch <= 2 ? sizeof(Ml1Warp<2>) : sizeof(Ml1Warp<4>));
    SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMThreads, smem));
    per_sm = a.blocks_per_sm > 0 ? std::min(std::max(per_sm, 1), a.blocks_per_sm) : 1;
    const int64_t items = a.seg_end - a.seg_begin;
    int64_t grid = (items + (kMThreads / 32) - 1) / (kMThreads / 32);
    grid = std::min<int64_t>(grid, (int64_t)per_sm * sm_count());
    if (grid >= 1) {
      kern<<<(unsigned)grid, kMThreads, smem, s>>>(a);
      count_launch();
      SFG_CUDA(cudaGetLastError());
    }
    return;
  }
  switch (a.S) {
  case 1:
    launch_s<1>(a, s);
    break;
  case 2:
    launch_s<2>(a, s);
    break;
  case 4:
    launch_s<4>(a, s);
    break;
  case 8:
    launch_s<8>(a, s);
    break;
  case 16:
    launch_s<16>(a, s);
    break;
  case 32:
    launch_s<32>(a, s);
    break;
  default:
    throw InvalidArgument("nsys must be a power of two <= 32");
  }
}

} // namespace sfg
