// Batched subdomain-local OpInf replay for the regularisation selection (
// P:L725-729, grid P:L808; reading R34).
//
// Every candidate model b (one per lambda of the grid) is an OpInf ROM with its own operator
// O_b = [-Kbar | Bbar | -Hbar | -Cbar]; it is advanced alone with explicit Newmark over the K steps of
// the training run, driven by the training run's reduced Schwarz data g^_k, and scored by
//     err_b = ||Ubar - U^hat_b||_F / ||Ubar||_F      (reduced coordinates).
// One block per model, persistent over the K steps (the steps of one model are sequential; the
// models are independent): state u^, v^, a^ in shared memory, z = [u~; g^_k; u~^*2; u~^*3] and O_b
// (row-major) in shared memory when they fit (else z in a per-model global row, O_b from L2).  The
// step is latency-bound, so a warp works on 4 output rows at once (4 independent FMA chains per
// lane, interleaved warp sums) and the block has 16 warps.  Error partials stay with the lane that
// owns a row and are reduced in a fixed order at the end.
#include "osam_internal.h"

namespace osam {

namespace {

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

constexpr int RT = 512;
constexpr int RW = RT / 32;
constexpr int RROWS = 4;  // rows per warp in flight

// z[0:r] = u (already there), features z[r + r_b + q] = prod u[idx[q][.]]
__device__ __forceinline__ void features(const ReplayArgs& A, const double* u, double* z) {
  for (int q = threadIdx.x; q < A.nf; q += RT) {
    const int i = A.feat_idx[3 * q], j = A.feat_idx[3 * q + 1], l = A.feat_idx[3 * q + 2];
    double v = u[i] * u[j];
    if (l >= 0) v *= u[l];
    z[A.r + A.r_b + q] = v;
  }
}

// out[i] = O_b[i, :] z  for the rows owned by this warp (i = w + RW (RROWS g + q)); calls f(i, value)
// on lane 0.  Row ownership is fixed, so every sum has a fixed order.
template <class F>
__device__ __forceinline__ void matvec(const ReplayArgs& A, const double* Ob, const double* z, F f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rz = A.r + A.r_b + A.nf;
  for (int i0 = w; i0 < A.r; i0 += RW * RROWS) {
    double acc[RROWS];
    const double* row[RROWS];
#pragma unroll
    for (int q = 0; q < RROWS; ++q) {
      acc[q] = 0.0;
      const int i = i0 + q * RW;
      row[q] = Ob + (long long)(i < A.r ? i : i0) * rz;
    }
    for (int j = lane; j < rz; j += 32) {
      const double zj = z[j];
#pragma unroll
      for (int q = 0; q < RROWS; ++q) acc[q] = fma(row[q][j], zj, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < RROWS; ++q) acc[q] = warp_sum(acc[q]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < RROWS; ++q)
        if (i0 + q * RW < A.r) f(i0 + q * RW, acc[q]);
  }
}

__global__ void __launch_bounds__(RT) replay_kernel(const ReplayArgs A) {
  extern __shared__ double sm[];
  const int b = blockIdx.x, r = A.r;
  double* u = sm;
  double* v = sm + r;
  double* a = sm + 2 * r;
  __shared__ double red[2][RW];
  const int rz = r + A.r_b + A.nf;
  const double* Ob = A.O + (long long)b * r * rz;
  double* z = A.z_in_smem ? sm + 3 * r : A.z + (long long)b * rz;
  if (A.o_in_smem) {  // stage O_b once (it is read every step)
    double* Os = sm + 3 * r + rz;
    for (long long t = threadIdx.x; t < (long long)r * rz; t += RT) Os[t] = Ob[t];
    Ob = Os;
  }
  double* traj = A.traj ? A.traj + (long long)b * A.K * r : nullptr;
  const double dt = A.dt, c2 = 0.5 * A.dt * A.dt;
  // step 0: u^_0 = Ubar[:, 0], v^_0, a^_0 = O_b z_0
  for (int i = threadIdx.x; i < r; i += RT) {
    u[i] = A.Ubar[i];
    v[i] = A.vh0 ? A.vh0[i] : 0.0;
    z[i] = u[i];
    if (traj) traj[i] = u[i];
  }
  for (int j = threadIdx.x; j < A.r_b; j += RT) z[r + j] = A.Ghat[j];
  __syncthreads();
  features(A, u, z);
  __syncthreads();
  double num = 0.0, den = 0.0;  // lane-0 partials of the rows this warp owns
  matvec(A, Ob, z, [&](int i, double an) {
    a[i] = an;
    const double ub = A.Ubar[i];
    den = fma(ub, ub, den);
  });
  __syncthreads();
  for (int k = 1; k < A.K; ++k) {
    for (int i = threadIdx.x; i < r; i += RT) {
      const double ut = fma(c2, a[i], fma(dt, v[i], u[i]));
      u[i] = ut;
      z[i] = ut;
    }
    for (int j = threadIdx.x; j < A.r_b; j += RT) z[r + j] = A.Ghat[(long long)k * A.r_b + j];
    __syncthreads();
    features(A, u, z);
    __syncthreads();
    matvec(A, Ob, z, [&](int i, double an) {
      v[i] = fma(0.5 * dt, a[i] + an, v[i]);
      a[i] = an;
      const double ub = A.Ubar[(long long)k * r + i];
      const double e = ub - u[i];
      num = fma(e, e, num);
      den = fma(ub, ub, den);
      if (traj) traj[(long long)k * r + i] = u[i];
    });
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][w] = num;
    red[1][w] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double n = 0.0, d = 0.0;
    for (int q = 0; q < RW; ++q) {
      n += red[0][q];
      d += red[1][q];
    }
    A.err[b] = sqrt(n) / sqrt(d);
  }
}

// O column-major r x rz per model -> row-major
__global__ void transpose_ops_kernel(int r, int rz, int B, const double* __restrict__ in, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long per = (long long)r * rz;
  if (t >= per * B) return;
  const long long b = t / per, e = t % per;
  const long long i = e / rz, j = e % rz;  // out[b][i][j]
  out[t] = in[b * per + i + (long long)r * j];
}

// first argmin over the finite errors (-1: none finite)
__global__ void argmin_kernel(int B, const double* __restrict__ err, int* __restrict__ best) {
  int k = -1;
  for (int b = 0; b < B; ++b)
    if (isfinite(err[b]) && (k < 0 || err[b] < err[k])) k = b;
  *best = k;
}

}  // namespace

void launch_transpose_ops(int r, int rz, int B, const double* in, double* out, cudaStream_t s) {
  transpose_ops_kernel<<<cdiv((long long)r * rz * B, 256), 256, 0, s>>>(r, rz, B, in, out);
  debug_check("transpose_ops_kernel", s);
}

cudaError_t launch_replay(ReplayArgs A, cudaStream_t s) {
  const size_t rz = (size_t)A.r + A.r_b + A.nf;
  constexpr size_t SMEM_MAX = 200 * 1024;
  size_t smem = sizeof(double) * 3 * (size_t)A.r;
  A.z_in_smem = smem + sizeof(double) * rz <= SMEM_MAX;
  if (A.z_in_smem) smem += sizeof(double) * rz;
  A.o_in_smem = A.z_in_smem && smem + sizeof(double) * rz * A.r <= SMEM_MAX;
  if (A.o_in_smem) smem += sizeof(double) * rz * A.r;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  replay_kernel<<<A.B, RT, smem, s>>>(A);
  debug_check("replay_kernel", s);
  argmin_kernel<<<1, 1, 0, s>>>(A.B, A.err, A.best);
  debug_check("argmin_kernel", s);
  return cudaGetLastError();
}

}  // namespace osam
