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
};

// One block: a 32 x 32 tile of C over the K range [z kc, (z+1) kc): A and B staged once in shared
// memory, then 2 x 2 m8n8k4 fragments per warp accumulate over k in increasing order.
__global__ void __launch_bounds__(128) dmma_gemm_kernel(const GemmArgs g) {
  pdl_enter();
  __shared__ double As[KMAX][TM + 1];  // As[k][m]
  __shared__ double Bs[KMAX][TN + 1];  // Bs[k][n]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN, k0 = blockIdx.z * g.kc;
  const int kn = min(g.kc, g.K - k0);
  for (int q = t; q < g.kc * TM; q += 128) {
    const int kk = q / TM, mm = q % TM;
    const int m = m0 + mm;
    As[kk][mm] = (m < g.M && kk < kn) ? g.A[m * g.sam + (k0 + kk) * g.sak] : 0.0;
  }
  for (int q = t; q < g.kc * TN; q += 128) {
    const int kk = q / TN, nn = q % TN;
    const int n = n0 + nn;
    Bs[kk][nn] = (n < g.N && kk < kn) ? g.B[(k0 + kk) * g.sbk + n * g.sbn] : 0.0;
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
  // no programmatic early launch for the GEMM: its many CTAs would sit on SMs the predecessors need
  dmma_gemm_kernel<<<dim3(dim3(cdiv(g.M, TM), cdiv(g.N, TN), cdiv(g.K, g.kc))), 128, 0, s>>>(g);
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

}  // namespace

// Batched ROM advance (B >= 2) on the tensor cores; scratch Z ((r + r_b) x B) and `part` (split-K
// partials, tc_part_size doubles).
long long tc_part_size(int r, int r_b, int nf, int B, long long n_s, long long n_lift3) {
  const long long a = (long long)gemm_splits(r, B, r + r_b + nf) * r * B;
  const long long g = r_b > 0 ? (long long)gemm_splits(r_b, B, (int)n_s) * r_b * B : 0;
  const long long l = n_lift3 > 0 ? (long long)gemm_splits((int)n_lift3, B, r) * n_lift3 * B : 0;
  return std::max(std::max(a, g), std::max<long long>(l, 1));
}

void launch_rom_advance_tc(const RomLaunch& L, const double* KB, double* Z, double* part, cudaStream_t s,
                           int* launches) {
  const int r = L.r, rb = L.r_b, rz = L.r + L.r_b + L.nf, B = L.B;
  launch_k(tc_predict_kernel, dim3(cdiv((long long)r * B, 256)), dim3(256), 0, s, r, rz, B, L.uh0, L.vh0, L.ah0, L.dt, L.c2, Z);
  debug_check("tc_predict_kernel", s);
  launch_rom_features(L.nf, B, L.feat_idx, Z, rz, Z + r + rb, rz, s);  // polynomial OpInf rows of Z
  *launches += L.nf > 0;
  if (rb > 0 && L.G) {  // folded exchange: g^ = G u^_src -> Z[r:, :]
    const int S = gemm(GemmArgs{rb, B, L.Gr, L.G, 1, rb, L.Gu, 1, L.Gr, nullptr, 0}, part, s);
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
  *launches += 3;
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

}  // namespace osam
