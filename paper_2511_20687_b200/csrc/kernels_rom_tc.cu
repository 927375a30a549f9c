// Batched OpInf ROM step on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64): the reduced update of
// the multi-sample configuration is a dense contraction (north_star (5)):
//
//   g^   = Phi_dS^T s                          (r_b x n_s) (n_s x B)
//   a^'  = e_b o ([-Kbar | Bbar] [u^*; g^])    (r x (r + r_b)) ((r + r_b) x B) (reading R22)
//   lift = Phi[donor rows] u^*                 (3 n_lift x r) (r x B)
//
// One generic kernel computes C = A B with arbitrary element strides (so transposes are free), a
// 32 x 32 C tile per block of 4 warps (16 x 16 per warp = 2 x 2 m8n8 fragments), split over K so that
// the small products of this config still cover the SMs; each block stages its K range of A and B in
// shared memory once.  The split-K partials are summed in split order by the consumer kernel: every C
// element accumulates in a fixed order and results are bitwise repeatable.  Tensor cores only here; the FOM path is HBM-bound and stays on the FP64 pipe.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "osam_internal.h"

namespace osam {

namespace {

constexpr int TM = 32, TN = 32, KMAX = 64;  // C tile per block, K range per block (split-K)

// D = A B + C for one m8n8k4 fp64 fragment: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// c/d = C[lane/4][2 (lane%4) + {0, 1}]  (PTX ISA, mma.m8n8k4 .f64).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct GemmArgs {
  int M, N, K;
  const double* A;
  long long sam, sak;  // A(m, k) = A[m sam + k sak]
  const double* B;
  long long sbk, sbn;  // B(k, n) = B[k sbk + n sbn]
  double* C;           // partial products: C[z][m + M n] for K split z (dense, M x N per split)
  int kc;              // K range of one split (multiple of 4, <= KMAX)
  const double* B2;    // rows k >= kb of B come from B2: B(k, n) = B2[(k - kb) sbk2 + n sbn2] (null: none)
  long long sbk2, sbn2;
  int kb;
};

// One block: a 32 x 32 tile of C over the K range [z kc, (z+1) kc): A and B staged once in shared
// memory, then 2 x 2 m8n8k4 fragments per warp accumulate over k in increasing order.
__global__ void __launch_bounds__(128) dmma_gemm_kernel(const GemmArgs g) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double As[KMAX][TM + 1];  // As[k][m]
  __shared__ double Bs[KMAX][TN + 1];  // Bs[k][n]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN, k0 = blockIdx.z * g.kc;
  const int kn = min(g.kc, g.K - k0);
  // A is an operator fixed at bind ([-Kbar | Bbar], the folded G, Phi_dS^T, Phi_lift): staged before waiting for
  // the predecessors (programmatic dependent launch); B is this sweep's data.  Each thread first loads all its
  // elements into registers (every load in flight at once; a load-then-store loop is a chain of L2 round trips),
  // consecutive threads along the operand's contiguous dimension, then stores them to shared memory.
  constexpr int PT = KMAX * TM / 128;
  static_assert(KMAX * TN / 128 == PT, "tile shapes");
  const bool a_mfast = g.sam == 1 || g.sak != 1;  // A contiguous in m (else in k)
  const bool b_kfast = g.sbk == 1 || g.sbn != 1;  // B contiguous in k (else in n)
  auto split = [&](int q, bool first_fast, int w, int& kk, int& x) {  // q -> (kk, m or n)
    if (first_fast) {
      kk = q / w;
      x = q - kk * w;
    } else {
      x = q / g.kc;
      kk = q - x * g.kc;
    }
  };
  double va[PT];
#pragma unroll
  for (int u = 0; u < PT; ++u) {
    const int q = t + 128 * u;
    double v = 0.0;
    if (q < g.kc * TM) {
      int kk, mm;
      split(q, a_mfast, TM, kk, mm);
      const int m = m0 + mm;
      if (m < g.M && kk < kn) v = g.A[m * g.sam + (k0 + kk) * g.sak];
    }
    va[u] = v;
  }
#pragma unroll
  for (int u = 0; u < PT; ++u) {
    const int q = t + 128 * u;
    if (q < g.kc * TM) {
      int kk, mm;
      split(q, a_mfast, TM, kk, mm);
      As[kk][mm] = va[u];
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int u = 0; u < PT; ++u) {
    const int q = t + 128 * u;
    double v = 0.0;
    if (q < g.kc * TN) {
      int kk, nn;
      split(q, !b_kfast, TN, kk, nn);
      const int n = n0 + nn;
      const int k = k0 + kk;
      if (n < g.N && kk < kn)
        v = (g.B2 && k >= g.kb) ? g.B2[(k - g.kb) * g.sbk2 + n * g.sbn2] : g.B[k * g.sbk + n * g.sbn];
    }
    va[u] = v;
  }
#pragma unroll
  for (int u = 0; u < PT; ++u) {
    const int q = t + 128 * u;
    if (q < g.kc * TN) {
      int kk, nn;
      split(q, !b_kfast, TN, kk, nn);
      Bs[kk][nn] = va[u];
    }
  }
  __syncthreads();
  const int wm = (warp & 1) * 16, wn = (warp >> 1) * 16;  // warp sub-tile
  double acc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  for (int ks = 0; ks < g.kc; ks += 4) {
    double a[2], b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = As[ks + (lane & 3)][wm + 8 * i + (lane >> 2)];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = Bs[ks + (lane & 3)][wn + 8 * j + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double* C = g.C + (size_t)blockIdx.z * g.M * g.N;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (m < g.M && n < g.N) C[m + (long long)g.M * n] = acc[i][j][h];
      }
}

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// number of K splits: enough blocks to cover the SMs, K range <= KMAX
int gemm_splits(int M, int N, int K) {
  const long long tiles = (long long)cdiv(M, TM) * cdiv(N, TN);
  long long s = std::max<long long>(cdiv(K, KMAX), cdiv(296, tiles));
  s = std::min<long long>(s, cdiv(K, 4));
  return (int)std::max<long long>(1, s);
}

// C partials for S = gemm_splits(M, N, K) splits into `part` (S x M x N doubles); returns S.
int gemm(GemmArgs g, double* part, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return 0;
  const int S = gemm_splits(g.M, g.N, g.K);
  g.kc = (int)(cdiv(cdiv(g.K, S), 4) * 4);
  g.C = part;
  // programmatic early launch (OSAM_GEMM_PDL=1): the CTAs stage A while the predecessors finish; measured
  // against the plain launch (its many CTAs may sit on SMs the predecessors need)
  static const bool gemm_pdl = getenv("OSAM_GEMM_PDL") && getenv("OSAM_GEMM_PDL")[0] == '1';
  const dim3 grid(cdiv(g.M, TM), cdiv(g.N, TN), cdiv(g.K, g.kc));
  if (gemm_pdl)
    launch_k(dmma_gemm_kernel, grid, dim3(128), 0, s, g);
  else
    dmma_gemm_kernel<<<grid, 128, 0, s>>>(g);
  debug_check("dmma_gemm_kernel", s);
  return (int)cdiv(g.K, g.kc);
}

// C(m, n) = sum_z part[z][m + M n] in split order, into a strided destination
__global__ void reduce_splits_kernel(int M, int N, int S, const double* __restrict__ part, double* __restrict__ C,
                                     long long scm, long long scn) {
  pdl_enter();
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= (long long)M * N) return;
  double v = 0.0;
  for (int z = 0; z < S; ++z) v += part[(size_t)z * M * N + q];
  C[(q % M) * scm + (q / M) * scn] = v;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Z[0:r, b] = u~ = u^ + dt v^ + c2 a^   (Z is rz x B, column-major; c2 = dt^2/2 explicit)
__global__ void tc_predict_kernel(int r, int rz, int B, const double* __restrict__ uh, const double* __restrict__ vh,
                                  const double* __restrict__ ah, double dt, double c2, double* __restrict__ Z) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= r * B) return;
  const int i = t % r, b = t / r;
  Z[i + (long long)rz * b] = fma(c2, ah[t], fma(dt, vh[t], uh[t]));
}

// a^' = e_b * araw, v^' = v^ + dt/2 (a^ + a^'), u^' = u^*, norm partials (active samples only).
// grid (ceil(r/256), B); partial layout [slot][B] with slot = blockIdx.x.  mode 1: a^ only (all
// samples); mode 2: implicit right-hand side e_b * araw into ah1 (active samples), rom_implicit_kernel
// finishes.
__global__ void __launch_bounds__(256) tc_epilogue_kernel(const RomLaunch L, const double* __restrict__ part,
                                                          int S, const double* __restrict__ Z, int rz, int mode) {
  pdl_enter();
  __shared__ double red[2][8];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  const int r = L.r;
  const bool on = i < r && (mode == 1 || L.active[b]);
  double num = 0.0, den = 0.0;
  if (on) {
    const long long id = i + (long long)r * b;
    double araw = 0.0;
    for (int z = 0; z < S; ++z) araw += part[(size_t)z * r * L.B + id];  // split-K partials, fixed order
    const double an = L.e[b] * araw;
    if (mode != 0) {
      L.ah1[id] = an;
    } else {
      const double un = Z[i + (long long)rz * b];
      const double vn = fma(0.5 * L.dt, L.ah0[id] + an, L.vh0[id]);
      if (L.with_norm) {
        const double d = (un - L.uh1[id]) + L.dt * (vn - L.vh1[id]);
        const double w = un + L.dt * vn;
        num = d * d;
        den = w * w;
      }
      L.uh1[id] = un;
      L.vh1[id] = vn;
      L.ah1[id] = an;
    }
  }
  if (mode != 0) return;
  num = warp_sum(num);
  den = warp_sum(den);
  const int t = threadIdx.x;
  if ((t & 31) == 0) {
    red[0][t >> 5] = num;
    red[1][t >> 5] = den;
  }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, c = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += red[0][w];
      c += red[1][w];
    }
    L.partial[(long long)blockIdx.x * L.B + b] = make_double2(a, c);
  }
}

// lift = sum of the split-K partials; rows that are Schwarz DOFs take the ROM's own s
// (Dirichlet rows: Phi_lift row is zero)
__global__ void tc_lift_reduce_kernel(long long nl, int B, int S, const double* __restrict__ part,
                                      const int* __restrict__ code, const double* __restrict__ s, long long ns,
                                      double* __restrict__ out) {
  pdl_enter();
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (q >= nl) return;
  const int cd = code[q];
  double v = 0.0;
  if (cd <= -2) {
    v = s[(long long)b * ns + (-2 - cd)];
  } else {
    for (int z = 0; z < S; ++z) v += part[(size_t)z * nl * B + (long long)b * nl + q];
  }
  out[(long long)b * nl + q] = v;
}


// ---- persistent controller for batched tensor-core ROM groups (osam_internal.h RomPArgs) -------------------
__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// One C tile (TM x TN over K split z) by the 128 threads t of one half of the CTA (named barrier bid): the body
// of dmma_gemm_kernel.
__device__ void gemm_tile_dev(const GemmArgs& g, int mt, int nt, int z, double (*As)[TM + 1], double (*Bs)[TN + 1],
                              int t, int bid) {
  const int lane = t & 31, warp = t >> 5;
  const int m0 = mt * TM, n0 = nt * TN, k0 = z * g.kc;
  const int kn = min(g.kc, g.K - k0);
  bar_named(bid, 128);  // the previous tile of this half is done with As, Bs
  for (int q = t; q < g.kc * TM; q += 128) {
    const int kk = q / TM, mm = q % TM;
    const int m = m0 + mm;
    As[kk][mm] = (m < g.M && kk < kn) ? g.A[m * g.sam + (k0 + kk) * g.sak] : 0.0;
  }
  for (int q = t; q < g.kc * TN; q += 128) {
    const int kk = q / TN, nn = q % TN;
    const int n = n0 + nn;
    const int k = k0 + kk;
    Bs[kk][nn] = (n < g.N && kk < kn)
                     ? ((g.B2 && k >= g.kb) ? g.B2[(k - g.kb) * g.sbk2 + n * g.sbn2] : g.B[k * g.sbk + n * g.sbn])
                     : 0.0;
  }
  bar_named(bid, 128);
  const int wm = (warp & 1) * 16, wn = (warp >> 1) * 16;
  double acc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  for (int ks = 0; ks < g.kc; ks += 4) {
    double a[2], b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = As[ks + (lane & 3)][wm + 8 * i + (lane >> 2)];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = Bs[ks + (lane & 3)][wn + 8 * j + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double* C = g.C + (size_t)z * g.M * g.N;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (m < g.M && n < g.N) C[m + (long long)g.M * n] = acc[i][j][h];
      }
}

constexpr int RP_T = 256;  // threads of the persistent CTA (two 128-thread GEMM halves)

// Grid-wide barrier of the co-resident CTAs (cooperative launch): one arrival counter and a generation word in
// global memory; thread 0 of each CTA arrives with a release fence and waits with acquire loads (nanosleep
// backoff), the last arrival resets the counter and publishes the next generation.  bar[0] count, bar[1] gen.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire_gpu(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      st_release_gpu(bar + 1, g + 1);
    } else {
      while (ld_acquire_gpu(bar + 1) == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}



__device__ __forceinline__ void rom_step_begin(const Ctl& C, int B) {
  for (int b = 0; b < B; ++b) {
    C.active[b] = 1;
    C.iters[b] = 0;
  }
  C.flags[0] = 1;
  C.flags[1] = 0;
  *C.n_dev = 0;
  *C.step_dev += 1;
}

__global__ void __launch_bounds__(RP_T) rom_persistent_kernel(const __grid_constant__ RomPArgs A) {
  extern __shared__ __align__(16) unsigned char rp_smem[];
  auto As = reinterpret_cast<double (*)[KMAX][TM + 1]>(rp_smem);
  auto Bs = reinterpret_cast<double (*)[KMAX][TN + 1]>(rp_smem + 2 * sizeof(double) * KMAX * (TM + 1));
  __shared__ double red[2][RP_T / 32];
  const Ctl& C = A.ctl;
  const int B = A.B;
  const int t = threadIdx.x, lane = t & 31;
  for (int k = 0; k < A.n_steps; ++k) {
    if (blockIdx.x == 0 && t == 0) rom_step_begin(C, B);
    grid_barrier(A.bar);
    for (int n = 1; n <= A.max_iters; ++n) {
      const bool first = n == 1;
      for (int i = 0; i < A.n_sd; ++i) {
        const RomPSub& d = A.s[i];
        const RomPSub& src = A.s[d.src];
        const int c = (k & 1) ? 1 - d.cur0 : d.cur0;
        const int cs = (k & 1) ? 1 - src.cur0 : src.cur0;
        const bool newest = (d.src < i) || !first;  // iterate n of an earlier source, else n - 1 (n = 1: checkpoint)
        // phase 1: predictor u~ -> Z[0:r] (as tc_predict_kernel) and the folded boundary input g^ = G u^_src
        // -> Z[r:r+rb], one warp per (row, sample): lane l sums k = l, l + 32, ... in order, then a butterfly
        for (int q = blockIdx.x * RP_T + t; q < d.r * B; q += gridDim.x * RP_T) {
          const int ii = q % d.r, b = q / d.r;
          d.Z[ii + (long long)d.rz * b] = fma(A.c2, d.rst[c][2][q], fma(A.dt, d.rst[c][1][q], d.rst[c][0][q]));
        }
        {
          const double* Gu = src.rst[newest ? 1 - cs : cs][0];
          for (int q = (blockIdx.x * RP_T + t) >> 5; q < d.rb * B; q += (gridDim.x * RP_T) >> 5) {
            const int m = q % d.rb, b = q / d.rb;
            const double* gr = d.G + m;
            const double* ub = Gu + (long long)d.Gr * b;
            double v = 0.0;
#pragma unroll 4
            for (int kk = lane; kk < d.Gr; kk += 32) v = fma(gr[(long long)d.rb * kk], ub[kk], v);
            v = warp_sum(v);
            if (lane == 0) d.Z[d.r + m + (long long)d.rz * b] = v;
          }
        }
        grid_barrier(A.bar);
        // phase 2: araw = [-Kbar | Bbar] [u~; g^], split-K DMMA tiles (the plan of gemm()), two per CTA at a time
        {
          GemmArgs g{d.r, B, d.rz, d.KB, 1, d.r, d.Z, 1, d.rz, d.part, d.kc_u};
          const int mt_n = (d.r + TM - 1) / TM, nt_n = (B + TN - 1) / TN;
          const int tasks = mt_n * nt_n * d.S_u;
          const int half = t >> 7, th = t & 127;
          for (int q = 2 * blockIdx.x + half; q < tasks; q += 2 * gridDim.x) {
            const int z = q % d.S_u, tile = q / d.S_u;
            gemm_tile_dev(g, tile % mt_n, tile / mt_n, z, As[half], Bs[half], th, 1 + half);
          }
        }
        grid_barrier(A.bar);
        // phase 3: epilogue (tc_epilogue_kernel, mode 0): a^', v^', u^', norm partials of the active samples
        const int nblk = (d.r + RP_T - 1) / RP_T;
        for (int u = blockIdx.x; u < nblk * B; u += gridDim.x) {
          const int blk = u % nblk, b = u / nblk;
          const int ii = blk * RP_T + t;
          double num = 0.0, den = 0.0;
          if (ii < d.r && C.active[b]) {
            const long long id = ii + (long long)d.r * b;
            double araw = 0.0;
            for (int z = 0; z < d.S_u; ++z) araw += __ldcg(d.part + (size_t)z * d.r * B + id);
            const double an = d.e[b] * araw;
            const double un = d.Z[ii + (long long)d.rz * b];
            const double vn = fma(0.5 * A.dt, d.rst[c][2][id] + an, d.rst[c][1][id]);
            if (!first) {
              const double dd = (un - d.rst[1 - c][0][id]) + A.dt * (vn - d.rst[1 - c][1][id]);
              const double w = un + A.dt * vn;
              num = dd * dd;
              den = w * w;
            }
            d.rst[1 - c][0][id] = un;
            d.rst[1 - c][1][id] = vn;
            d.rst[1 - c][2][id] = an;
          }
          num = warp_sum(num);
          den = warp_sum(den);
          if (lane == 0) {
            red[0][t >> 5] = num;
            red[1][t >> 5] = den;
          }
          __syncthreads();
          if (t == 0) {
            double a = 0.0, cc = 0.0;
            for (int w = 0; w < RP_T / 32; ++w) {
              a += red[0][w];
              cc += red[1][w];
            }
            A.partial[(long long)(d.slot0 + blk) * B + b] = make_double2(a, cc);
          }
          __syncthreads();
        }
        grid_barrier(A.bar);
      }
      // K3, per sample (CTA b, warp 0): finalize_kernel's fixed-order sum (1024 virtual threads: thread v holds
      // slot v, a warp butterfly per 32, the warp sums added in order; virtual warps beyond the slots add +0.0 and
      // are skipped, exactly), the test and the sample's flags
      for (int b = blockIdx.x; b < B; b += gridDim.x) {
        if (t < 32) {
          double num = 0.0, den = 0.0;
          if (n >= A.min_iters)
            for (int w = 0; 32 * w < A.n_slots; ++w) {
              const int v = 32 * w + lane;
              double x = 0.0, y = 0.0;
              if (v < A.n_slots) {
                const double2 pv = __ldcg(A.partial + (long long)v * B + b);
                x = pv.x;
                y = pv.y;
              }
              num += warp_sum(x);
              den += warp_sum(y);
            }
          if (lane == 0 && C.active[b]) {
            C.iters[b] = n;
            if (C.iters_all) C.iters_all[(long long)(*C.step_dev - 1) * B + b] = n;
            if (n >= A.min_iters) {
              C.numden[2 * b] = num;
              C.numden[2 * b + 1] = den;
              if (C.trace && n <= C.trace_T) {
                double* tr = C.trace + 2 * (((long long)(*C.step_dev - 1) * C.trace_T + (n - 1)) * B + b);
                tr[0] = num;
                tr[1] = den;
              }
              if (!isfinite(num) || !isfinite(den)) {
                C.flags[1] = 1;
                C.sticky[0] = 1;
              }
              bool conv = (num == 0.0) || (num < A.tol_rel * A.tol_rel * den);
              if (A.tol_abs > 0.0) conv = conv || (num < A.tol_abs * A.tol_abs);
              if (conv) C.active[b] = 0;
            }
          }
        }
      }
      grid_barrier(A.bar);
      // the continue decision, in every CTA from the same flags (nothing writes them until the next barrier)
      int any = 0;
      for (int b = t; b < B; b += RP_T) any |= __ldcg(C.active + b);
      any = __syncthreads_or(any);
      const bool unstable = __ldcg(C.flags + 1) != 0;
      const bool go = any && !unstable && n < A.max_iters;
      if (blockIdx.x == 0 && t == 0) {  // any_active_body's bookkeeping
        *C.n_dev = n;
        C.flags[0] = any;
        if (any && n >= A.max_iters) C.sticky[1] = 1;
      }
      if (!go) break;
    }
    grid_barrier(A.bar);  // every CTA has read this step's flags before block 0 begins the next step
  }
}

}  // namespace

// Batched ROM advance (B >= 2) on the tensor cores; scratch Z ((r + r_b) x B) and `part` (split-K
// partials, tc_part_size doubles).
long long tc_gemm_part(int M, int N, int K) { return (long long)gemm_splits(M, N, K) * M * N; }

long long tc_part_size(int r, int r_b, int nf, int B, long long n_s, long long n_lift3) {
  const long long a = (long long)gemm_splits(r, B, r + r_b + nf) * r * B;
  const long long g = r_b > 0 ? (long long)gemm_splits(r_b, B, (int)n_s) * r_b * B : 0;
  const long long l = n_lift3 > 0 ? (long long)gemm_splits((int)n_lift3, B, r) * n_lift3 * B : 0;
  return std::max(std::max(a, g), std::max<long long>(l, 1));
}

int launch_rom_update_gemm_tc(const RomLaunch& L, double* Z, double* part, cudaStream_t s, int* launches) {
  const int r = L.r, rz = L.r + L.r_b + L.nf, B = L.B;
  GemmArgs ga{r, B, r + L.Gr, L.KBG, 1, r, Z, 1, rz, nullptr, 0, L.Gu, 1, L.Gld ? L.Gld : L.Gr, r};
  ++*launches;
  return gemm(ga, part, s);
}

void launch_rom_predict_tc(const RomLaunch& L, double* Z, cudaStream_t s, int* launches) {
  const int r = L.r, rb = L.r_b, rz = L.r + L.r_b + L.nf, B = L.B;
  launch_k(tc_predict_kernel, dim3(cdiv((long long)r * B, 256)), dim3(256), 0, s, r, rz, B, L.uh0, L.vh0, L.ah0, L.dt, L.c2, Z);
  debug_check("tc_predict_kernel", s);
  launch_rom_features(L.nf, B, L.feat_idx, Z, rz, Z + r + rb, rz, s);  // polynomial OpInf rows of Z
  *launches += 1 + (L.nf > 0);
}

void launch_rom_advance_tc(const RomLaunch& L, const double* KB, double* Z, double* part, cudaStream_t s,
                           int* launches) {
  const int r = L.r, rb = L.r_b, rz = L.r + L.r_b + L.nf, B = L.B;
  if (!L.pre) {
    launch_rom_predict_tc(L, Z, s, launches);
    --*launches;  // counted with the advance below
  }
  if (L.pre && L.KBG) {  // araw = [-Kbar | Bbar G] [u~; u^_src]: the exchange folded into the update (one GEMM)
    GemmArgs ga{r, B, r + L.Gr, L.KBG, 1, r, Z, 1, rz, nullptr, 0, L.Gu, 1, L.Gld ? L.Gld : L.Gr, r};
    const int S = gemm(ga, part, s);
    launch_k(tc_epilogue_kernel, dim3(dim3(cdiv(r, 256), B)), dim3(256), 0, s, L, part, S, Z, rz, 0);
    debug_check("tc_epilogue_kernel", s);
    *launches += 2;
    return;
  }
  if (rb > 0 && L.G) {  // folded exchange: g^ = G u^_src -> Z[r:, :]
    const int S = gemm(GemmArgs{rb, B, L.Gr, L.G, 1, rb, L.Gu, 1, L.Gld ? L.Gld : L.Gr, nullptr, 0}, part, s);
    launch_k(reduce_splits_kernel, dim3(cdiv((long long)rb * B, 256)), dim3(256), 0, s, rb, B, S, part, Z + r, 1, rz);
    debug_check("reduce_splits_kernel", s);
    *launches += 2;
  } else if (rb > 0) {  // g^ = Phi_dS^T s  -> Z[r:, :]
    const int S = gemm(GemmArgs{rb, B, (int)L.n_sdof, L.Phi_s, L.n_sdof, 1, L.s, 1, L.n_sdof, nullptr, 0}, part, s);
    launch_k(reduce_splits_kernel, dim3(cdiv((long long)rb * B, 256)), dim3(256), 0, s, rb, B, S, part, Z + r, 1, rz);
    debug_check("reduce_splits_kernel", s);
    *launches += 2;
  }
  if (L.beta > 0.0 && L.nf > 0) {  // implicit polynomial ROM: Newton per sample on u~ = Z[0:r], g^ = Z[r:]
    launch_rom_newton(L, Z, rz, Z + r, rz, 0, rom_partial_slots(r, true), s);
    *launches += 2;
    return;
  }
  // araw = [-Kbar | Bbar] Z, reduced in the epilogue
  const int S = gemm(GemmArgs{r, B, rz, KB, 1, r, Z, 1, rz, nullptr, 0}, part, s);
  launch_k(tc_epilogue_kernel, dim3(dim3(cdiv(r, 256), B)), dim3(256), 0, s, L, part, S, Z, rz, L.beta > 0.0 ? 2 : 0);
  debug_check("tc_epilogue_kernel", s);
  *launches += L.pre ? 2 : 3;
  if (L.beta > 0.0) {
    launch_rom_implicit(L, Z, rz, rom_partial_slots(r, true), s);
    ++*launches;
  }
}

// Initial acceleration a^0 = e (-Kbar u^0 + Bbar Phi_dS^T s0) on the same path.
void launch_rom_accel_tc(const RomLaunch& L, const double* uh, double* ah, const double* KB, double* Z, double* part,
                         cudaStream_t s, int* launches) {
  const int r = L.r, rb = L.r_b, rz = L.r + L.r_b + L.nf, B = L.B;
  RomLaunch A = L;
  A.ah1 = ah;
  launch_k(tc_predict_kernel, dim3(cdiv((long long)r * B, 256)), dim3(256), 0, s, r, rz, B, uh, uh, uh, 0.0, 0.0, Z);  // Z[0:r] = u^0
  debug_check("tc_predict_kernel", s);
  launch_rom_features(L.nf, B, L.feat_idx, Z, rz, Z + r + rb, rz, s);
  *launches += L.nf > 0;
  if (rb > 0) {
    const int S = gemm(GemmArgs{rb, B, (int)L.n_sdof, L.Phi_s, L.n_sdof, 1, L.s, 1, L.n_sdof, nullptr, 0}, part, s);
    launch_k(reduce_splits_kernel, dim3(cdiv((long long)rb * B, 256)), dim3(256), 0, s, rb, B, S, part, Z + r, 1, rz);
    debug_check("reduce_splits_kernel", s);
    *launches += 2;
  }
  const int S = gemm(GemmArgs{r, B, rz, KB, 1, r, Z, 1, rz, nullptr, 0}, part, s);
  launch_k(tc_epilogue_kernel, dim3(dim3(cdiv(r, 256), B)), dim3(256), 0, s, A, part, S, Z, rz, 1);
  debug_check("tc_epilogue_kernel", s);
  *launches += 3;
}

// lift = Phi_lift u^ (all 3 n_lift rows; non-free rows of Phi_lift are zero), Schwarz rows := s.
void launch_rom_lift_tc(int r, int B, long long nl, const double* Phi_lift, const int* code, const double* uh,
                        const double* sv, long long ns, double* out, double* part, cudaStream_t st, int* launches) {
  if (nl == 0) return;
  const int S = gemm(GemmArgs{(int)nl, B, r, Phi_lift, r, 1, uh, 1, r, nullptr, 0}, part, st);
  launch_k(tc_lift_reduce_kernel, dim3(dim3(cdiv(nl, 256), B)), dim3(256), 0, st, nl, B, S, part, code, sv, ns, out);
  debug_check("tc_lift_reduce_kernel", st);
  *launches += 2;
}


void rom_persist_plan(int r, int rb, int Gr, int B, RomPSub* p) {
  auto plan = [](int M, int N, int K, int* S, int* kc) {
    const int s = gemm_splits(M, N, K);
    *kc = (int)(cdiv(cdiv(K, s), 4) * 4);
    *S = (int)cdiv(K, *kc);
  };
  plan(r, B, r + rb, &p->S_u, &p->kc_u);
  (void)Gr;
}

int rom_persist_slots(int r) { return (int)cdiv(r, TM); }
int rom_persist_tiles(int r, int B) { return (int)(cdiv(r, TM) * cdiv(B, TN)); }

cudaError_t launch_rom_persistent(const RomPArgs& A, cudaStream_t s) {
  const size_t smem = 2 * sizeof(double) * KMAX * (TM + 1) + 2 * sizeof(double) * KMAX * (TN + 1);
  static int grid = 0;
  if (grid == 0) {
    cudaFuncSetAttribute(rom_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rom_persistent_kernel, RP_T, smem);
    grid = std::max(1, sms * std::min(1, std::max(1, per_sm)));  // one CTA per SM (two GEMM tiles at a time)
  }
  int g = grid;
  if (const char* e = getenv("OSAM_ROM_PERSIST_GRID")) g = std::max(1, std::min(grid, atoi(e)));
  void* args[] = {const_cast<RomPArgs*>(&A)};
  return cudaLaunchCooperativeKernel((void*)rom_persistent_kernel, dim3(g), dim3(RP_T), args, smem, s);
}

}  // namespace osam
