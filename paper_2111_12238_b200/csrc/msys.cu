// msys.cu -- batched solve executor with one chain per lane (combos 1 and 8,
// S >= 2 systems; SFG_EXECUTOR=msys).
//
// A warp owns a group of 32 consecutive chains (the B = 32 layout of the
// multi-line executor, mline.cuh) and one PAIR of the batch's systems: work
// item = (group, pair), and a group's pairs are consecutive tickets.  Lane b
// advances chain b one row per step; in-group dependencies come from a
// shared-memory ring, everything else is staged ahead:
//
//   record   (row, dependency codes)       cp.async 16 B, kDR steps ahead
//   values   (one pre-arranged record)     cp.async 16 B, kDV steps ahead
//   x words  (external dependencies, rhs)  cp.async 16 B, kDX steps ahead
//
// (optionally the record and values are prefetched HBM -> L2 further ahead,
// SFG_MSYS_PF steps beyond kDR).  Measured on config 5 this executor is
// slower than the chain executor -- see DESIGN.md section 4 -- and stays an
// opt-in ablation.
//
// Each row's dependencies (reference summation order) are split at inspection
// into an EARLY prefix that holds only external dependencies and a LATE
// suffix of at most LCH terms that holds every ring dependency.  The early
// partial sum of step i+1 is formed while step i is still in flight, so a
// step's critical path is: ring values -> LCH products -> carry -> division.
// Padding is exact: padded slots multiply a zero value by a zero word, and
// acc - (+0) == acc for every acc, so the sums equal the reference's
// sequential trsv_csr_row (kernels.hpp:173-177) bit for bit.
#include "common.cuh"
#include "mline.cuh"

#include <algorithm>

namespace sfg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kDR = 5, kDV = 3, kDX = 3;
constexpr int kQR = kDR + 1, kQV = kDV + 1, kQX = kDX + 1;

__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// 16-byte copy with zero fill: bytes = 0 writes zeros and reads nothing
__device__ __forceinline__ void cp16z(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(dst)), "l"(src),
               "r"(bytes));
}
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ bool sent2(unsigned long long a, unsigned long long b) {
  return is_sent_hi(a) || is_sent_hi(b);
}

template <int ECH, int LCH> struct Shape {
  static constexpr int NE = ECH + LCH;
  static constexpr int NV = NE + 3;                // value pairs per record
  static constexpr int RW = (2 + NE + 3) / 4 * 4;  // record int32 (16-byte multiple)
};

template <int ECH, int LCH> struct alignas(16) MsWarp {
  using K = Shape<ECH, LCH>;
  int32_t rec[kQR][32][K::RW];
  double v[kQV][32][K::NV][2];
  unsigned long long x[kQX][32][K::NE][2];
  unsigned long long rhs[kQX][32][2];
  double ring[kRing][32][2];
};

template <int ECH, int LCH>
__global__ void __launch_bounds__(32) k_msys(const MLineArgs A) {
  using K = Shape<ECH, LCH>;
  constexpr int NE = K::NE, NV = K::NV, RW = K::RW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MsWarp<ECH, LCH>& W = *reinterpret_cast<MsWarp<ECH, LCH>*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int S = A.S;
  const int NP = S / 2;
  uint32_t uR = 0, uV = 0; // steps staged so far: the record / value slot of a step
  const int64_t total = (int64_t)(A.seg_end - A.seg_begin) * NP;
  for (;;) {
    unsigned long long w0 = 0;
    if (lane == 0)
      w0 = atomicAdd(A.counter, 1ull);
    const long long wi = (long long)__shfl_sync(FULL, w0, 0);
    if (wi >= total)
      break;
    const int item = A.seg_begin + (int)(wi / NP);
    const int pair = (int)(wi % NP);
    const int s0 = 2 * pair;
    const bool second = item >= A.f_ngroup;
    const bool bwd = second && A.combo == 8;
    const int32_t* mrec = bwd ? A.b_mrec : A.f_mrec;
    const double* mval = (bwd ? A.b_mval : A.f_mval) + (size_t)pair * A.n * (NV * 2);
    const int32_t* cstart = bwd ? A.b_cstart : A.f_cstart;
    const int32_t* cskew = bwd ? A.b_cskew : A.f_cskew;
    const int nchain = bwd ? A.b_nchain : A.f_nchain;
    const int g = second ? __ldg((bwd ? A.b_gorder : A.f_gorder) + (item - A.f_ngroup))
                         : __ldg(A.f_gorder + item);
    const int T = __ldg((bwd ? A.b_gsteps : A.f_gsteps) + g);
    const int c = g * 32 + lane;
    const bool has_chain = c < nchain;
    const int p0 = has_chain ? __ldg(cstart + c) : 0;
    const int len = has_chain ? __ldg(cstart + c + 1) - p0 : 0;
    const int skew = has_chain ? __ldg(cskew + c) : 0;
    double* xo = second ? A.vout : A.vmid;
    const double* rhs_vec = second ? A.vmid : A.vin;
    const int kern = second ? 2 : 1;
    const uint32_t bR = uR, bV = uV;
    uR += T;
    uV += T;
    auto act = [&](int j) {
      const int o = j - skew;
      return o >= 0 && o < len && j < T;
    };
    double carry0 = 0.0, carry1 = 0.0, part0 = 0.0, part1 = 0.0;
    unsigned long long tr_claim = 0, tr_first = 0, poll_cyc = 0, late_cyc = 0;
    if (A.trace)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_claim));
    __syncwarp();
#pragma unroll 1
    for (int i = -kDR; i < T; ++i) {
      if (A.trace && i == 0)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_first));
      // cp.async groups of iterations <= i-2 complete: records of steps <=
      // i+kDR-2, values, x words and rhs of steps <= i+1
      wait_group<1>();
      __syncwarp();
      { // ---- record of step i + kDR
        const int j = i + kDR;
        if (j >= 0 && act(j)) {
          const int32_t* src = mrec + (int64_t)(p0 + j - skew) * RW;
          int32_t* dst = W.rec[(bR + j) % kQR][lane];
#pragma unroll
          for (int h = 0; h < RW; h += 4)
            cp16z(dst + h, src + h, 16u);
        }
      }
      if (A.lookahead > 0) { // ---- HBM -> L2 prefetch of the record and values of step i + PF
        const int j = i + kDR + A.lookahead;
        if (j >= 0 && act(j)) {
          prefetch_l2(mrec + (int64_t)(p0 + j - skew) * RW, RW * 4);
          prefetch_l2(mval + (size_t)(p0 + j - skew) * (NV * 2), NV * 16);
        }
      }
      { // ---- values of step i + kDV
        const int j = i + kDV;
        if (j >= 0 && act(j)) {
          const double* src = mval + (size_t)(p0 + j - skew) * (NV * 2);
          double* dst = &W.v[(bV + j) % kQV][lane][0][0];
#pragma unroll
          for (int h = 0; h < NV; ++h)
            cp16z(dst + 2 * h, src + 2 * h, 16u);
        }
      }
      { // ---- external x words and rhs of step i + kDX
        const int j = i + kDX;
        if (j >= 0 && j < T) {
          const uint32_t u = bR + j;
          if (act(j)) {
            const int32_t* R = W.rec[u % kQR][lane];
            const int fl = R[1];
            const int ne = (fl >> 8) & 0xff, nl = (fl >> 16) & 0xff;
            const int q = j % kQX;
#pragma unroll
            for (int a = 0; a < ECH; ++a) {
              const bool ok = a < ne;
              cp16z(&W.x[q][lane][a][0], xo + (size_t)(ok ? R[2 + a] : 0) * S + s0, ok ? 16u : 0u);
            }
#pragma unroll
            for (int a = 0; a < LCH; ++a) {
              const int cd = R[2 + ECH + a];
              const bool ok = a < nl && cd >= 0;
              cp16z(&W.x[q][lane][ECH + a][0], xo + (size_t)(ok ? cd : 0) * S + s0, ok ? 16u : 0u);
            }
            cp16z(&W.rhs[q][lane][0], rhs_vec + (size_t)R[0] * S + s0, 16u);
          }
        }
      }
      commit();
      // ---- late part of step i: ring terms, carry, division
      if (i >= 0 && act(i)) {
        const int32_t* R = W.rec[(bR + i) % kQR][lane];
        const double(*V)[2] = W.v[(bV + i) % kQV][lane];
        const int q = i % kQX;
        const int r = R[0];
        const int nl = (R[1] >> 16) & 0xff;
        unsigned long long l0[LCH > 0 ? LCH : 1], l1[LCH > 0 ? LCH : 1];
        bool ext_pending = false;
#pragma unroll
        for (int a = 0; a < LCH; ++a) {
          const int cd = R[2 + ECH + a];
          if (a < nl && cd < 0) {
            const int t = -1 - cd;
            const double* rg = W.ring[(i - (t >> 5)) & (kRing - 1)][t & 31];
            l0[a] = (unsigned long long)__double_as_longlong(rg[0]);
            l1[a] = (unsigned long long)__double_as_longlong(rg[1]);
          } else {
            l0[a] = W.x[q][lane][ECH + a][0];
            l1[a] = W.x[q][lane][ECH + a][1];
            ext_pending |= sent2(l0[a], l1[a]);
          }
        }
        if (__builtin_expect(ext_pending, 0)) {
#pragma unroll
          for (int a = 0; a < LCH; ++a) {
            const int cd = R[2 + ECH + a];
            if (a < nl && cd >= 0) {
              l0[a] = (unsigned long long)__double_as_longlong(poll_f64(xo + (size_t)cd * S + s0, 0));
              l1[a] = (unsigned long long)__double_as_longlong(
                  poll_f64(xo + (size_t)cd * S + s0 + 1, 0));
            }
          }
          if (A.trace)
            poll_cyc += 1;
        }
        double acc0 = part0, acc1 = part1;
#pragma unroll
        for (int a = 0; a < LCH; ++a) {
          acc0 = __dsub_rn(acc0, __dmul_rn(V[ECH + a][0], __longlong_as_double((long long)l0[a])));
          acc1 = __dsub_rn(acc1, __dmul_rn(V[ECH + a][1], __longlong_as_double((long long)l1[a])));
        }
        acc0 = __dsub_rn(acc0, __dmul_rn(V[NE][0], carry0));
        acc1 = __dsub_rn(acc1, __dmul_rn(V[NE][1], carry1));
        const double d0 = V[NE + 1][0], d1 = V[NE + 1][1];
        if (d0 == 0.0 || d1 == 0.0)
          report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
        const double x0 = div_with_rcp(acc0, d0, V[NE + 2][0]);
        const double x1 = div_with_rcp(acc1, d1, V[NE + 2][1]);
        publish_f64(xo + (size_t)r * S + s0, x0);
        publish_f64(xo + (size_t)r * S + s0 + 1, x1);
        W.ring[i & (kRing - 1)][lane][0] = x0;
        W.ring[i & (kRing - 1)][lane][1] = x1;
        carry0 = x0;
        carry1 = x1;
      }
      // ---- early part of step i+1: rhs minus the external prefix
      if (i + 1 >= 0 && act(i + 1)) {
        const int j = i + 1;
        const int32_t* R = W.rec[(bR + j) % kQR][lane];
        const double(*V)[2] = W.v[(bV + j) % kQV][lane];
        const int q = j % kQX;
        unsigned long long e0[ECH], e1[ECH];
        unsigned long long r0w = W.rhs[q][lane][0], r1w = W.rhs[q][lane][1];
        bool pending = sent2(r0w, r1w);
#pragma unroll
        for (int a = 0; a < ECH; ++a) {
          e0[a] = W.x[q][lane][a][0];
          e1[a] = W.x[q][lane][a][1];
          pending |= sent2(e0[a], e1[a]);
        }
        if (__builtin_expect(pending, 0)) {
          const int ne = (R[1] >> 8) & 0xff;
          const double* rp = rhs_vec + (size_t)R[0] * S + s0;
          if (sent2(r0w, r1w)) {
            r0w = (unsigned long long)__double_as_longlong(poll_f64(rp, A.sleep_ns));
            r1w = (unsigned long long)__double_as_longlong(poll_f64(rp + 1, A.sleep_ns));
          }
#pragma unroll
          for (int a = 0; a < ECH; ++a)
            if (a < ne && sent2(e0[a], e1[a])) {
              const double* xp = xo + (size_t)R[2 + a] * S + s0;
              e0[a] = (unsigned long long)__double_as_longlong(poll_f64(xp, A.sleep_ns));
              e1[a] = (unsigned long long)__double_as_longlong(poll_f64(xp + 1, A.sleep_ns));
            }
          if (A.trace)
            poll_cyc += 1;
        }
        double acc0 = __longlong_as_double((long long)r0w);
        double acc1 = __longlong_as_double((long long)r1w);
#pragma unroll
        for (int a = 0; a < ECH; ++a) {
          acc0 = __dsub_rn(acc0, __dmul_rn(V[a][0], __longlong_as_double((long long)e0[a])));
          acc1 = __dsub_rn(acc1, __dmul_rn(V[a][1], __longlong_as_double((long long)e1[a])));
        }
        part0 = acc0;
        part1 = acc1;
      }
      __syncwarp();
    }
    wait_group<0>();
    __syncwarp();
    if (A.trace) {
      unsigned long long pm = poll_cyc;
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) {
        const unsigned long long v = __shfl_xor_sync(FULL, pm, o2);
        pm = v > pm ? v : pm;
      }
      if (lane == 0) {
        unsigned long long te;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        unsigned long long* tr = A.trace + (size_t)wi * 4;
        tr[0] = tr_claim;
        tr[1] = tr_first;
        tr[2] = te;
        tr[3] = (late_cyc << 32) | (pm & 0xffffffffull);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// inspector
// ---------------------------------------------------------------------------
inline unsigned grid_of(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * 32;
  g = g > cap ? cap : g;
  return (unsigned)(g < 1 ? 1 : g);
}

// per position: non-carry dependency count and the length of the suffix that
// starts at the first ring dependency (0 if none)
__global__ void msys_split_kernel(const int32_t* __restrict__ ptr, int32_t n, int dir,
                                  const int32_t* __restrict__ cstart,
                                  const int32_t* __restrict__ chain_of,
                                  const int32_t* __restrict__ code, int* stats) {
  int nd_max = 0, late_max = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const bool chained = (int)p > cstart[chain_of[p]];
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int e0 = ptr[r], nd = ptr[r + 1] - e0 - 1 - (chained ? 1 : 0);
    int fr = nd;
    for (int a = nd - 1; a >= 0; --a)
      if (code[e0 + a] < 0)
        fr = a;
    nd_max = nd > nd_max ? nd : nd_max;
    late_max = nd - fr > late_max ? nd - fr : late_max;
  }
  atomicMax(&stats[0], nd_max);
  atomicMax(&stats[1], late_max);
}

__global__ void msys_rec_kernel(const int32_t* __restrict__ ptr, int32_t n, int dir,
                                const int32_t* __restrict__ cstart,
                                const int32_t* __restrict__ chain_of,
                                const int32_t* __restrict__ code, int ech, int lch, int rw,
                                int32_t* __restrict__ rec) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const bool chained = (int)p > cstart[chain_of[p]];
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int e0 = ptr[r], nd = ptr[r + 1] - e0 - 1 - (chained ? 1 : 0);
    const int ne = nd > lch ? nd - lch : 0; // early count
    const int nl = nd - ne;
    int32_t* R = rec + p * rw;
    R[0] = r;
    R[1] = (chained ? 1 : 0) | (ne << 8) | (nl << 16);
    for (int a = 0; a < ech; ++a)
      R[2 + a] = a < ne ? code[e0 + a] : 0;
    for (int a = 0; a < lch; ++a)
      R[2 + ech + a] = a < nl ? code[e0 + ne + a] : 0;
    for (int a = 2 + ech + lch; a < rw; ++a)
      R[a] = 0;
  }
}

// per (position, pair): {early values, late values, carry coefficient,
// diagonal, RN(1/diagonal)} for the pair's two systems, zero padded
__global__ void msys_val_kernel(const int32_t* __restrict__ ptr, const double* __restrict__ val,
                                int32_t n, int dir, int32_t S, const int32_t* __restrict__ rec,
                                int ech, int lch, int rw, double* __restrict__ mval) {
  const int NV = ech + lch + 3;
  const int NP = S / 2;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * NP;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t % n;
    const int pair = (int)(t / n);
    const int32_t* R = rec + p * rw;
    const int r = R[0];
    const bool chained = (R[1] & 1) != 0;
    const int ne = (R[1] >> 8) & 0xff, nl = (R[1] >> 16) & 0xff;
    const int e0 = ptr[r], e1 = ptr[r + 1];
    double* out = mval + ((size_t)pair * n + p) * (NV * 2);
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * pair + h;
      for (int a = 0; a < ech; ++a)
        out[a * 2 + h] = a < ne ? val[(size_t)(e0 + a) * S + s] : 0.0;
      for (int a = 0; a < lch; ++a)
        out[(ech + a) * 2 + h] = a < nl ? val[(size_t)(e0 + ne + a) * S + s] : 0.0;
      out[(ech + lch) * 2 + h] = chained ? val[(size_t)(e1 - 2) * S + s] : 0.0;
      const double d = val[(size_t)(e1 - 1) * S + s];
      out[(ech + lch + 1) * 2 + h] = d;
      out[(ech + lch + 2) * 2 + h] = __drcp_rn(d);
    }
  }
}

struct ShapeChoice {
  int ech, lch;
};
constexpr ShapeChoice kShapes[] = {{4, 2}, {9, 3}, {12, 4}};

template <int ECH, int LCH> void launch_shape(const MLineArgs& a, cudaStream_t s) {
  auto kern = k_msys<ECH, LCH>;
  const size_t smem = sizeof(MsWarp<ECH, LCH>);
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem));
  per_sm = std::max(per_sm, 1);
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  const int64_t items = (int64_t)(a.seg_end - a.seg_begin) * (a.S / 2);
  int64_t grid = std::min<int64_t>(items, (int64_t)per_sm * sm_count());
  if (const char* e = getenv("SFG_MSYS_GRID"))
    grid = std::min<int64_t>(grid, std::max(1, atoi(e)));
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, 32, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

} // namespace

bool build_msys(const int32_t* ptr, const double* val, int32_t n, int dir, int32_t S,
                MLineLayout& L, cudaStream_t s) {
  if (L.B != 32 || S < 2 || S % 2 != 0 || n == 0)
    return false;
  DBuf<int> stats(2);
  SFG_CUDA(cudaMemsetAsync(stats.p, 0, 2 * sizeof(int), s));
  msys_split_kernel<<<grid_of(n), 256, 0, s>>>(ptr, n, dir, L.cstart.p, L.chain_of.p, L.code.p,
                                               stats.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  int h[2] = {0, 0};
  SFG_CUDA(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  const int nd_max = h[0], late_max = h[1];
  int ech = -1, lch = -1;
  for (const ShapeChoice& c : kShapes)
    if (c.lch >= late_max && c.ech + c.lch >= nd_max) {
      ech = c.ech;
      lch = c.lch;
      break;
    }
  if (ech < 0)
    return false;
  L.ech = ech;
  L.lch = lch;
  L.mrec_w = (2 + ech + lch + 3) / 4 * 4;
  L.mrec.alloc((int64_t)n * L.mrec_w);
  msys_rec_kernel<<<grid_of(n), 256, 0, s>>>(ptr, n, dir, L.cstart.p, L.chain_of.p, L.code.p, ech,
                                             lch, L.mrec_w, L.mrec.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  L.mval.alloc((int64_t)n * (S / 2) * (ech + lch + 3) * 2);
  refresh_msys_values(ptr, val, n, dir, S, L, s);
  return true;
}

void refresh_msys_values(const int32_t* ptr, const double* val, int32_t n, int dir, int32_t S,
                         MLineLayout& L, cudaStream_t s) {
  if (!L.mval.p)
    return;
  msys_val_kernel<<<grid_of((int64_t)n * (S / 2)), 256, 0, s>>>(ptr, val, n, dir, S, L.mrec.p,
                                                                L.ech, L.lch, L.mrec_w, L.mval.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void launch_msys(const MLineArgs& a, cudaStream_t s) {
  if (a.ech == 4 && a.lch == 2)
    launch_shape<4, 2>(a, s);
  else if (a.ech == 9 && a.lch == 3)
    launch_shape<9, 3>(a, s);
  else if (a.ech == 12 && a.lch == 4)
    launch_shape<12, 4>(a, s);
  else
    throw InvalidArgument("k_msys: no record shape instantiated for this split");
}

} // namespace sfg
