// K2 Schwarz transfer, K3 convergence finalisation, and the OpInf ROM kernels (K4-K6).
//
// K2  s[p, c] = sum_{b<8} w_pb U_src[idx_pb, c],  w_pb = prod_d (xi_d or 1 - xi_d)
//     pointwise (trilinear) projection Pi of the source's current field onto the
//     destination's Schwarz nodes (reading R11).
// K3  num = sum_slots num_slot, den = sum_slots den_slot in a fixed order; converged iff
//     n >= min_iters and (num == 0 or num < tol_rel^2 den or num < tol_abs^2)
//     (eq:conv_criterion P:L443-467; readings R6, R7, R29).
// K4  g^ = Phi_dS^T s
// K5  u^* = u^ + dt v^ + dt^2/2 a^ ; a^' = e_b(-Kbar u^* + Bbar g^) ; v^' = v^ + dt/2 (a^ + a^')
//     plus reduced-coordinate norm partials (reading R8)  (P:L617-722 eq:schwarz_opinf_discrete)
// K6  lift at donor nodes: Phi[donor rows] u^* (free), 0 (Dirichlet), own s (Schwarz)
#include <algorithm>

#include "osam_internal.h"

namespace osam {

namespace {

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// compact = 1: write dst[b][3p + c] (a trace slot) instead of dst[b][out[3p + c]].  One thread per
// (node, component): the gather is memory-latency-bound (a y-z slab of an x-fastest field), so more
// independent loads in flight matter more than sharing the weights.
__global__ void transfer_kernel(int n, const int* __restrict__ idx, const double* __restrict__ xi,
                                const int* __restrict__ out, const double* __restrict__ src, long long cs,
                                long long bs_src, double* __restrict__ dst, long long bs_dst,
                                const int* __restrict__ active, int compact) {
  // The map (out, xi, idx) is fixed at bind, so it is read before waiting for the predecessor (programmatic
  // dependent launch): only the source field and the store depend on earlier kernels of the sweep.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  const bool in = t < 3 * n;
  const int p = in ? t / 3 : 0, c = in ? t - 3 * p : 0;
  const int o = in ? out[3 * p + c] : -1;
  double x = 0.0, y = 0.0, z = 0.0;
  int id[8];
  if (o >= 0) {
    x = xi[3 * p];
    y = xi[3 * p + 1];
    z = xi[3 * p + 2];
#pragma unroll
    for (int q = 0; q < 8; ++q) id[q] = idx[8 * p + q];
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (o < 0 || (active != nullptr && !active[b])) return;
  const double* sb = src + b * bs_src + c * cs;
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double w = ((q & 1) ? x : 1.0 - x) * ((q & 2) ? y : 1.0 - y) * ((q & 4) ? z : 1.0 - z);
    acc = fma(w, sb[id[q]], acc);
  }
  dst[b * bs_dst + (compact ? 3 * p + c : o)] = acc;
}

// Xi (reading R31): s = (1 - alpha) T[lo] + alpha T[lo + 1] from the trace slots of one map
__global__ void trace_interp_kernel(int n, const int* __restrict__ out, const double* __restrict__ trace,
                                    long long slot_stride, int lo, double alpha, double* __restrict__ dst,
                                    long long bs_dst, const int* __restrict__ active) {
  pdl_enter();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (p >= n || (active != nullptr && !active[b])) return;
  const double* T = trace + (long long)b * 3 * n + 3 * p;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int o = out[3 * p + c];
    if (o < 0) continue;
    double v = T[lo * slot_stride + c];
    if (alpha != 0.0) v = (1.0 - alpha) * v + alpha * T[(lo + 1) * slot_stride + c];
    dst[b * bs_dst + o] = v;
  }
}

__global__ void step_begin_kernel(Ctl c, int B) {
  pdl_enter();
  const int b = threadIdx.x;
  for (int q = b; q < B; q += blockDim.x) {
    c.active[q] = 1;
    c.iters[q] = 0;
  }
  if (b == 0) {
    c.flags[0] = 1;
    c.flags[1] = 0;
    *c.n_dev = 0;
    *c.step_dev += 1;
  }
}

// after finalize (single thread): n_dev += 1, flags[0] = any sample active, per-step iteration
// counts, max_iters flag, and (graph mode) the condition of the sweep while-loop
__device__ __forceinline__ void any_active_finish(const Ctl& c, int n, int a) {
  c.flags[0] = a;
  const bool more = a && n < c.max_iters && !c.flags[1];
  if (a && n >= c.max_iters) c.sticky[1] = 1;
  if (c.has_cond) cudaGraphSetConditional(c.cond, more ? 1u : 0u);
}

__device__ void any_active_stamps(const Ctl& c, int n);

// thread 0 of any_active_kernel after the block has folded the samples: n_dev, the K1 timeline, flags
__device__ __forceinline__ void any_active_tail(const Ctl& c, int a) {
  const int n = *c.n_dev + 1;
  *c.n_dev = n;
  if (c.stamps) any_active_stamps(c, n);
  any_active_finish(c, n, a);
}

__device__ __forceinline__ void any_active_body(const Ctl& c, int B) {
  const int n = *c.n_dev + 1;
  *c.n_dev = n;
  if (c.stamps) any_active_stamps(c, n);
  int a = 0;
  for (int b = 0; b < B; ++b) a |= c.active[b];
  if (c.iters_all) {
    const long long k = *c.step_dev - 1;
    for (int b = 0; b < B; ++b) c.iters_all[k * B + b] = c.iters[b];
  }
  any_active_finish(c, n, a);
}
// K1 timeline of the sweep that just ran (every K1 of the sweep joined before K3): union, sum and count of the
// subdomains' K1 intervals into busy[], stamps reset
__device__ void any_active_stamps(const Ctl& c, int n) {
  unsigned long long s[8], e[8];
  int m = 0;
  for (int i = 0; i < c.n_stamp && m < 8; ++i) {
    const unsigned long long a = c.stamps[2 * i], b = c.stamps[2 * i + 1];
    c.stamps[2 * i] = ~0ULL;
    c.stamps[2 * i + 1] = 0ULL;
    if (a == ~0ULL || b < a) continue;  // no K1 of subdomain i in this sweep
    int q = m++;
    for (; q > 0 && s[q - 1] > a; --q) {  // insertion sort by start
      s[q] = s[q - 1];
      e[q] = e[q - 1];
    }
    s[q] = a;
    e[q] = b;
  }
  double uni = 0.0, sum = 0.0;
  unsigned long long lo = 0, hi = 0;
  for (int q = 0; q < m; ++q) {
    sum += (double)(e[q] - s[q]);
    if (q == 0 || s[q] > hi) {
      if (q > 0) uni += (double)(hi - lo);
      lo = s[q];
      hi = e[q];
    } else if (e[q] > hi) {
      hi = e[q];
    }
  }
  if (m > 0) uni += (double)(hi - lo);
  c.busy[0] += uni;
  c.busy[1] += sum;
  c.busy[2] += m;
  c.busy[3] += 1.0;
  c.busy[4] += n >= 2 ? 1.0 : 0.0;
}



// B > 1: the per-sample parts of any_active_body spread over the block (a single thread walking B samples is a
// chain of L2 round trips: 9 us for c5's 64), then thread 0 finishes
__global__ void any_active_kernel(Ctl c, int B) {
  pdl_enter();
  __shared__ int any;
  const int t = threadIdx.x;
  if (t == 0) any = 0;
  __syncthreads();
  int a = 0;
  for (int b = t; b < B; b += blockDim.x) a |= c.active[b];
  if (a) any = 1;  // benign: every writer stores 1
  if (c.iters_all) {
    const long long k = *c.step_dev - 1;
    for (int b = t; b < B; b += blockDim.x) c.iters_all[k * B + b] = c.iters[b];
  }
  __syncthreads();
  if (t == 0) any_active_tail(c, any);
}

// one block of FIN_T threads per sample; the sweep that just ran is iteration n = *n_dev + 1.  fused
// (B = 1): thread 0 then runs any_active_body itself (every thread read n_dev before the barrier)
constexpr int FIN_T = 1024;
__global__ void __launch_bounds__(FIN_T) finalize_kernel(Ctl c, const double2* __restrict__ part, int n_slots, int B,
                                                         int min_iters, double tol_rel, double tol_abs, int fused) {
  pdl_enter();
  __shared__ double red[2][FIN_T / 32];
  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const int n = *c.n_dev + 1;
  double num = 0.0, den = 0.0;
  if (n >= min_iters) {
#pragma unroll 4
    for (int s = t; s < n_slots; s += blockDim.x) {
      const double2 v = part[(long long)s * B + b];
      num += v.x;
      den += v.y;
    }
  }
  num = warp_sum(num);
  den = warp_sum(den);
  if ((t & 31) == 0) {
    red[0][t >> 5] = num;
    red[1][t >> 5] = den;
  }
  __syncthreads();
  if (t == 0) {
    num = 0.0;
    den = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) {
      num += red[0][w];
      den += red[1][w];
    }
    if (c.active[b]) {
      c.iters[b] = n;
      if (n >= min_iters) {
        c.numden[2 * b] = num;
        c.numden[2 * b + 1] = den;
        if (c.trace && n <= c.trace_T) {  // convergence trace (osam_set_conv_trace)
          double* tr = c.trace + 2 * (((long long)(*c.step_dev - 1) * c.trace_T + (n - 1)) * B + b);
          tr[0] = num;
          tr[1] = den;
        }
        if (!isfinite(num) || !isfinite(den)) {
          c.flags[1] = 1;
          c.sticky[0] = 1;
        }
        bool conv = (num == 0.0) || (num < tol_rel * tol_rel * den);
        if (tol_abs > 0.0) conv = conv || (num < tol_abs * tol_abs);
        if (conv) c.active[b] = 0;
      }
    }
    if (fused) any_active_body(c, B);
  }
}


// Programmatic dependent launch, split: a kernel lets its dependents launch, reads what its predecessors do
// not write (operators and maps fixed at bind) and only then waits for them (pdl_enter does both at once).
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Fixed-order block sum of one value per thread (blockDim.x = 256).
__device__ __forceinline__ double block_sum256(double v) {
  __shared__ double red[8];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < 8; ++w) t += red[w];
  return t;
}

// Partial g^: gpart[z][b][k] = sum over chunk z of the Schwarz DOFs of Phi_s[q, k] s[q, b]
// (a block per (k, chunk, sample); thread-strided, fixed order).  The consumer sums the chunks in order.
constexpr int GCHUNK = 2048;
__global__ void __launch_bounds__(256) rom_project_bnd_kernel(int r_b, int B, long long ns,
                                                              const double* __restrict__ Phi_s,
                                                              const double* __restrict__ s,
                                                              double* __restrict__ gpart) {
  pdl_launch();
  const int k = blockIdx.x, z = blockIdx.y, b = blockIdx.z;
  const double* col = Phi_s + (long long)k * ns;
  const double* sb = s + (long long)b * ns;
  const long long q0 = (long long)z * GCHUNK, q1 = q0 + GCHUNK < ns ? q0 + GCHUNK : ns;
  constexpr int PER = GCHUNK / 256;
  double phi[PER];  // this thread's Phi_s entries, read before the wait (fixed at bind)
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const long long q = q0 + threadIdx.x + 256LL * m;
    phi[m] = q < q1 ? col[q] : 0.0;
  }
  pdl_wait();
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const long long q = q0 + threadIdx.x + 256LL * m;
    if (q < q1) acc = fma(phi[m], sb[q], acc);
  }
  acc = block_sum256(acc);
  if (threadIdx.x == 0) gpart[((long long)z * B + b) * r_b + k] = acc;
}

// u~ = u^ + dt v^ + c2 a^  (c2 = dt^2/2 explicit; dt^2 (1/2 - beta) implicit)
__global__ void rom_predict_kernel(int r, int B, const double* __restrict__ uh, const double* __restrict__ vh,
                                   const double* __restrict__ ah, double dt, double c2, double* __restrict__ us) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= r * B) return;
  us[t] = fma(c2, ah[t], fma(dt, vh[t], uh[t]));
}

// a^'[i,b] = e_b (sum_j KBr[i,j] z[j,b]), z = [u^*; g^], KBr = [-Kbar | Bbar] row-major; v^', norm
// partials.  A warp per output row (lanes stride the row: coalesced), 8 rows per block; the block's
// partial (num, den) sums its warps in order: grid (ceil(r/8), B), slot = blockIdx.x, layout [slot][B].
// mode 1: acceleration only (initial condition); mode 2 (implicit): the right-hand side
// e_b (-Kbar u~ + Bbar g^ ...) into ah1, finished by rom_implicit_kernel.
constexpr int UPD_GS_MAX = 1024;  // r_b staged in shared memory up to this (else per row, same order)
constexpr int UPD_PRE_K = 8, UPD_PRE_B = 2;  // row entries per lane read before the wait (r <= 256, r_b <= 64)
__global__ void __launch_bounds__(256) rom_update_kernel(const RomLaunch L, int mode) {
  pdl_launch();
  __shared__ double red[2][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 8 + w;
  const int b = blockIdx.y;
  const int r = L.r, rz = L.r + L.r_b + L.nf;
  // the operator row [-Kbar | Bbar] of this warp is fixed at bind: read it before waiting for the predecessors
  const bool pre = r <= 32 * UPD_PRE_K && L.r_b <= 32 * UPD_PRE_B && L.nf == 0 && i < r;
  double rk[UPD_PRE_K], rb_[UPD_PRE_B];
  if (pre) {
    const double* row = L.KBr + (long long)i * rz;
#pragma unroll
    for (int m = 0; m < UPD_PRE_K; ++m) rk[m] = lane + 32 * m < r ? row[lane + 32 * m] : 0.0;
#pragma unroll
    for (int m = 0; m < UPD_PRE_B; ++m) rb_[m] = lane + 32 * m < L.r_b ? row[r + lane + 32 * m] : 0.0;
  }
  pdl_wait();
  const bool on = i < r && (mode == 1 || L.active[b]);
  // g^[., b] = chunk partials summed in order, once per block (every row of the block reads it)
  __shared__ double gs[UPD_GS_MAX];
  const bool gsm = L.r_b <= UPD_GS_MAX;
  if (gsm) {
    for (int k = threadIdx.x; k < L.r_b; k += 256) {
      double g = 0.0;
      for (int z = 0; z < L.gchunks; ++z) g += L.gh[((long long)z * L.B + b) * L.r_b + k];
      gs[k] = g;
    }
    __syncthreads();
  }
  double num = 0.0, den = 0.0;
  if (on) {
    const double* row = L.KBr + (long long)i * rz;
    const double* us = L.ustar + (long long)r * b;
    double acc = 0.0;
    if (pre) {  // the same terms in the same order from the preloaded row
#pragma unroll
      for (int m = 0; m < UPD_PRE_K; ++m)
        if (lane + 32 * m < r) acc = fma(rk[m], us[lane + 32 * m], acc);
#pragma unroll
      for (int m = 0; m < UPD_PRE_B; ++m) {
        const int k = lane + 32 * m;
        if (k < L.r_b) {
          double g = 0.0;
          if (gsm)
            g = gs[k];
          else
            for (int z = 0; z < L.gchunks; ++z) g += L.gh[((long long)z * L.B + b) * L.r_b + k];
          acc = fma(rb_[m], g, acc);
        }
      }
    } else {
#pragma unroll 4
      for (int j = lane; j < r; j += 32) acc = fma(row[j], us[j], acc);
      for (int k = lane; k < L.r_b; k += 32) {
        double g = 0.0;  // g^[k, b]: chunk partials in order
        if (gsm)
          g = gs[k];
        else
          for (int z = 0; z < L.gchunks; ++z) g += L.gh[((long long)z * L.B + b) * L.r_b + k];
        acc = fma(row[r + k], g, acc);
      }
    }
    const double* fb = L.F + (long long)L.nf * b;  // polynomial OpInf features
    for (int q = lane; q < L.nf; q += 32) acc = fma(row[r + L.r_b + q], fb[q], acc);
    acc = warp_sum(acc);
    if (lane == 0) {
      const double an = L.e[b] * acc;
      const long long id = i + (long long)r * b;
      if (mode != 0) {  // acceleration only (initial condition) / implicit right-hand side
        L.ah1[id] = an;
      } else {
        const double vn = fma(0.5 * L.dt, L.ah0[id] + an, L.vh0[id]);
        const double un = us[i];
        if (L.with_norm) {
          const double d = (un - L.uh1[id]) + L.dt * (vn - L.vh1[id]);
          const double wv = un + L.dt * vn;
          num = d * d;
          den = wv * wv;
        }
        L.uh1[id] = un;
        L.vh1[id] = vn;
        L.ah1[id] = an;
      }
    }
  }
  if (mode != 0) return;
  if (lane == 0) {
    red[0][w] = num;
    red[1][w] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int q = 0; q < 8; ++q) {
      a += red[0][q];
      c += red[1][q];
    }
    L.partial[(long long)blockIdx.x * L.B + b] = make_double2(a, c);
  }
}

// out[b][ld] = code>=0 ? sum_j Phi_lift[ld, j] uh[j, b] : (code == -1 ? 0 : s[b][-2-code])
// A warp per LIFT_ROWS consecutive rows (their loads interleaved: more bytes in flight per warp, the
// read of Phi_lift is the HBM-relevant ROM traffic of c4), 16-byte loads when r is even; each row is
// summed per lane over j and then by the butterfly, as with one row per warp.
constexpr int LIFT_ROWS = 4;
__global__ void rom_lift_kernel(int r, int B, long long nl, const double* __restrict__ Phi_lift,
                                const int* __restrict__ code, const double* __restrict__ uh,
                                const double* __restrict__ s, long long ns, double* __restrict__ out) {
  pdl_launch();
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = (nl + LIFT_ROWS - 1) / LIFT_ROWS;  // warps per sample
  if (w >= nw * B) {
    pdl_wait();
    return;
  }
  const int b = (int)(w / nw);
  const long long ld0 = (w % nw) * LIFT_ROWS;
  int cd[LIFT_ROWS];
  const double* row[LIFT_ROWS];
  double acc[LIFT_ROWS];
#pragma unroll
  for (int q = 0; q < LIFT_ROWS; ++q) {
    cd[q] = ld0 + q < nl ? code[ld0 + q] : -1;
    row[q] = Phi_lift + (long long)(cd[q] >= 0 ? cd[q] : 0) * r;
    acc[q] = 0.0;
  }
  const double* u = uh + (long long)r * b;
  if ((r & 1) == 0 && r <= 256) {  // Phi_lift rows (fixed at bind) read before waiting for the predecessors
    double2 a[LIFT_ROWS][4];
#pragma unroll
    for (int q = 0; q < LIFT_ROWS; ++q)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        a[q][m] = (cd[q] >= 0 && lane + 32 * m < r / 2) ? reinterpret_cast<const double2*>(row[q])[lane + 32 * m]
                                                        : make_double2(0.0, 0.0);
    pdl_wait();
    const double2* u2 = reinterpret_cast<const double2*>(u);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int j = lane + 32 * m;
      if (j >= r / 2) break;
      const double2 x = u2[j];
#pragma unroll
      for (int q = 0; q < LIFT_ROWS; ++q)
        if (cd[q] >= 0) {
          acc[q] = fma(a[q][m].x, x.x, acc[q]);
          acc[q] = fma(a[q][m].y, x.y, acc[q]);
        }
    }
  } else if ((r & 1) == 0) {
    pdl_wait();
    const double2* u2 = reinterpret_cast<const double2*>(u);
#pragma unroll 2
    for (int j = lane; j < r / 2; j += 32) {
      const double2 x = u2[j];
#pragma unroll
      for (int q = 0; q < LIFT_ROWS; ++q)
        if (cd[q] >= 0) {
          const double2 a = reinterpret_cast<const double2*>(row[q])[j];
          acc[q] = fma(a.x, x.x, acc[q]);
          acc[q] = fma(a.y, x.y, acc[q]);
        }
    }
  } else {
    pdl_wait();
    for (int j = lane; j < r; j += 32) {
      const double x = u[j];
#pragma unroll
      for (int q = 0; q < LIFT_ROWS; ++q)
        if (cd[q] >= 0) acc[q] = fma(row[q][j], x, acc[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < LIFT_ROWS; ++q) {
    if (ld0 + q >= nl) break;
    double v = 0.0;
    if (cd[q] >= 0)
      v = warp_sum(acc[q]);
    else if (cd[q] <= -2)
      v = s[(long long)b * ns + (-2 - cd[q])];
    if (lane == 0) out[(long long)b * nl + ld0 + q] = v;
  }
}

// Projection onto the POD basis (IC only): part[z][b][i] = sum over row chunk z of
// Phi[q, i] field_b[dof(ids[q])]  (a block per (i, chunk, sample), thread-strided, fixed order), then
// out[i, b] = sum_z part[z][b][i] in chunk order.
constexpr int PCHUNK = 65536;
__global__ void __launch_bounds__(256) rom_project_kernel(long long nrows, int r, int B, const double* __restrict__ Phi,
                                                         const int* __restrict__ ids, const double* __restrict__ field,
                                                         long long fbs, long long n_nodes, double* __restrict__ part) {
  const int i = blockIdx.x, z = blockIdx.y, b = blockIdx.z;
  const double* col = Phi + (long long)i * nrows;
  const double* f = field + (long long)b * fbs;
  const long long q0 = (long long)z * PCHUNK, q1 = q0 + PCHUNK < nrows ? q0 + PCHUNK : nrows;
  double acc = 0.0;
  for (long long q = q0 + threadIdx.x; q < q1; q += 256) {
    const long long dof = ids[q];
    acc = fma(col[q], f[(dof % 3) * n_nodes + dof / 3], acc);
  }
  acc = block_sum256(acc);
  if (threadIdx.x == 0) part[((long long)z * B + b) * r + i] = acc;
}

__global__ void sum_chunks_kernel(int r, int B, int nz, const double* __restrict__ part, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= r * B) return;
  double v = 0.0;
  for (int z = 0; z < nz; ++z) v += part[(long long)z * r * B + t];
  out[t] = v;
}

// Implicit ROM (reading R32), one block per sample: a^' = Minv_b f (f = ah1 from rom_update mode 2),
// u^' = u~ + beta dt^2 a^', v^' = v^ + dt ((1 - gamma) a^ + gamma a^'), gamma = 1/2; norm partials in
// slot 0 of the sample (other slots 0).  ut: u~ with per-sample stride uts.
__global__ void __launch_bounds__(256) rom_implicit_kernel(const RomLaunch L, const double* __restrict__ ut,
                                                           long long uts, int n_slots) {
  pdl_enter();
  extern __shared__ double f[];
  const int b = blockIdx.x, r = L.r;
  if (!L.active[b]) return;
  for (int i = threadIdx.x; i < r; i += 256) f[i] = L.ah1[i + (long long)r * b];
  __syncthreads();
  const double* Mb = L.Minv + (long long)b * r * r;
  const double bdt2 = L.beta * L.dt * L.dt;
  double num = 0.0, den = 0.0;
  for (int i = threadIdx.x; i < r; i += 256) {
    double a = 0.0;
    for (int j = 0; j < r; ++j) a = fma(Mb[(long long)i * r + j], f[j], a);
    const long long id = i + (long long)r * b;
    const double un = fma(bdt2, a, ut[i + uts * b]);
    const double vn = L.vh0[id] + L.dt * (0.5 * L.ah0[id] + 0.5 * a);
    if (L.with_norm) {
      const double d = (un - L.uh1[id]) + L.dt * (vn - L.vh1[id]);
      const double w = un + L.dt * vn;
      num = fma(d, d, num);
      den = fma(w, w, den);
    }
    L.uh1[id] = un;
    L.vh1[id] = vn;
    L.ah1[id] = a;
  }
  const double tn = block_sum256(num);
  __syncthreads();
  const double td = block_sum256(den);
  if (threadIdx.x == 0) {
    L.partial[b] = make_double2(tn, td);
    for (int q = 1; q < n_slots; ++q) L.partial[(long long)q * L.B + b] = make_double2(0.0, 0.0);
  }
}

// Implicit polynomial ROM (reading R37), one block per active sample: Newton on
//   R(u) = u - u~ - beta dt^2 a(u),  a(u) = e_b O [u; g^; u^*2; u^*3],  O = [-Kbar | Bbar | -Hbar | -Cbar]
// from u = u~ + beta dt^2 a^, Jacobian I - beta dt^2 e_b (O_u + O_f dF/du) (each thread builds its own
// rows), Gauss-Jordan with partial pivoting in shared memory, until |du| <= 1e-14 |u| (<= 50 steps; a
// non-converged sample writes NaN into its norm partial -> OSAM_EUNSTABLE).  Then a^' = a(u^'),
// v^' = v^ + dt (a^ + a^')/2 and the norm partials (slot 0 of the sample, other slots 0).
// g^: gchunks > 0 -> chunk partials gsrc[(z B + b) r_b + j] summed in order (CUDA-core path), else
// gsrc[j + gstride b] (tensor-core path, Z rows).
__device__ __forceinline__ double newton_block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < 8; ++w) t += red[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(256) rom_newton_kernel(const RomLaunch L, const double* __restrict__ ut_all,
                                                         long long uts, const double* __restrict__ gsrc,
                                                         long long gstride, int gchunks, int n_slots) {
  pdl_enter();
  extern __shared__ double sm[];
  __shared__ double red[8];
  __shared__ int piv;
  const int b = blockIdx.x, r = L.r, rb = L.r_b, nf = L.nf, rz = r + rb + nf, t = threadIdx.x;
  if (!L.active[b]) return;
  double* u = sm;
  double* ut = u + r;
  double* g = ut + r;
  double* feat = g + rb;
  double* a = feat + nf;
  double* J = a + r;  // [r][r + 1]
  const int ld = r + 1;
  const double eb = L.e[b], c = L.beta * L.dt * L.dt;
  const long long off = (long long)r * b;
  for (int i = t; i < r; i += 256) {
    ut[i] = ut_all[i + uts * b];
    u[i] = fma(c, L.ah0[off + i], ut[i]);
  }
  for (int j = t; j < rb; j += 256) {
    double v = 0.0;
    if (gchunks > 0)
      for (int z = 0; z < gchunks; ++z) v += gsrc[((long long)z * L.B + b) * rb + j];
    else
      v = gsrc[j + gstride * b];
    g[j] = v;
  }
  __syncthreads();
  // a(u) into a[] (features of u first)
  auto accel = [&]() {
    for (int q = t; q < nf; q += 256) {
      const int i = L.feat_idx[3 * q], j = L.feat_idx[3 * q + 1], l = L.feat_idx[3 * q + 2];
      double v = u[i] * u[j];
      if (l >= 0) v *= u[l];
      feat[q] = v;
    }
    __syncthreads();
    const int lane = t & 31, w = t >> 5;
    for (int k = w; k < r; k += 8) {
      const double* row = L.KBr + (long long)k * rz;
      double acc = 0.0;
      for (int j = lane; j < rz; j += 32) acc = fma(row[j], j < r ? u[j] : (j < r + rb ? g[j - r] : feat[j - r - rb]), acc);
      acc = warp_sum(acc);
      if (lane == 0) a[k] = eb * acc;
    }
    __syncthreads();
  };
  bool converged = false;
  for (int it = 0; it < 50; ++it) {
    accel();
    // Jacobian rows and residual (thread k owns row k)
    for (int k = t; k < r; k += 256) {
      const double* row = L.KBr + (long long)k * rz;
      double* Jk = J + (long long)k * ld;
      for (int m = 0; m < r; ++m) Jk[m] = row[m];
      for (int q = 0; q < nf; ++q) {
        const double o = row[r + rb + q];
        const int i = L.feat_idx[3 * q], j = L.feat_idx[3 * q + 1], l = L.feat_idx[3 * q + 2];
        if (l < 0) {
          Jk[i] = fma(o, u[j], Jk[i]);
          Jk[j] = fma(o, u[i], Jk[j]);
        } else {
          Jk[i] = fma(o, u[j] * u[l], Jk[i]);
          Jk[j] = fma(o, u[i] * u[l], Jk[j]);
          Jk[l] = fma(o, u[i] * u[j], Jk[l]);
        }
      }
      for (int m = 0; m < r; ++m) Jk[m] = (m == k ? 1.0 : 0.0) - c * eb * Jk[m];
      Jk[r] = -(u[k] - ut[k] - c * a[k]);  // -R
    }
    __syncthreads();
    // Gauss-Jordan with partial pivoting on [J | -R]
    for (int k = 0; k < r; ++k) {
      if (t == 0) {
        int p = k;
        for (int i = k + 1; i < r; ++i)
          if (fabs(J[(long long)i * ld + k]) > fabs(J[(long long)p * ld + k])) p = i;
        piv = p;
      }
      __syncthreads();
      if (piv != k)
        for (int m = t; m < ld; m += 256) {
          const double tmp = J[(long long)k * ld + m];
          J[(long long)k * ld + m] = J[(long long)piv * ld + m];
          J[(long long)piv * ld + m] = tmp;
        }
      __syncthreads();
      const double inv = 1.0 / J[(long long)k * ld + k];
      __syncthreads();
      for (int m = t; m < ld; m += 256) J[(long long)k * ld + m] *= inv;
      __syncthreads();
      for (long long e = t; e < (long long)r * ld; e += 256) {
        const int i = (int)(e / ld), m = (int)(e % ld);
        if (i != k && m != k) J[e] = fma(-J[(long long)i * ld + k], J[(long long)k * ld + m], J[e]);
      }
      __syncthreads();
      for (int i = t; i < r; i += 256)
        if (i != k) J[(long long)i * ld + k] = 0.0;
      __syncthreads();
    }
    double du2 = 0.0, u2 = 0.0;
    for (int i = t; i < r; i += 256) {
      const double du = J[(long long)i * ld + r];
      u[i] += du;
      du2 = fma(du, du, du2);
      u2 = fma(u[i], u[i], u2);
    }
    const double sdu = newton_block_sum(du2, red), su = newton_block_sum(u2, red);
    if (sqrt(sdu) <= 1e-14 * sqrt(su)) {
      converged = true;
      break;
    }
  }
  accel();  // a^' = a(u^')
  double num = 0.0, den = 0.0;
  for (int i = t; i < r; i += 256) {
    const long long id = off + i;
    const double un = u[i], an = a[i];
    const double vn = L.vh0[id] + L.dt * (0.5 * L.ah0[id] + 0.5 * an);
    if (L.with_norm) {
      const double d = (un - L.uh1[id]) + L.dt * (vn - L.vh1[id]);
      const double w = un + L.dt * vn;
      num = fma(d, d, num);
      den = fma(w, w, den);
    }
    L.uh1[id] = un;
    L.vh1[id] = vn;
    L.ah1[id] = an;
  }
  const double tn = newton_block_sum(num, red), td = newton_block_sum(den, red);
  if (t == 0) {
    L.partial[b] = make_double2(converged ? tn : nan(""), td);
    for (int q = 1; q < n_slots; ++q) L.partial[(long long)q * L.B + b] = make_double2(0.0, 0.0);
  }
}

// Minv_b = (I + c e_b Kbar)^-1 (Kbar column-major): Gauss-Jordan with partial pivoting on [M | I],
// one block per sample (setup, once per dt_i).
__global__ void __launch_bounds__(256) rom_minv_kernel(int r, const double* __restrict__ Kbar,
                                                       const double* __restrict__ e, double c,
                                                       double* __restrict__ work, double* __restrict__ Minv) {
  extern __shared__ double fac[];
  __shared__ int piv;
  const int b = blockIdx.x, n2 = 2 * r;
  double* W = work + (long long)b * r * n2;
  const double ce = c * e[b];
  for (long long t = threadIdx.x; t < (long long)r * n2; t += 256) {
    const int i = (int)(t / n2), j = (int)(t % n2);
    W[t] = j < r ? (i == j ? 1.0 : 0.0) + ce * Kbar[i + (long long)r * j] : (j - r == i ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      for (int i = k + 1; i < r; ++i)
        if (fabs(W[(long long)i * n2 + k]) > fabs(W[(long long)p * n2 + k])) p = i;
      piv = p;
    }
    __syncthreads();
    if (piv != k)
      for (int j = threadIdx.x; j < n2; j += 256) {
        const double t = W[(long long)k * n2 + j];
        W[(long long)k * n2 + j] = W[(long long)piv * n2 + j];
        W[(long long)piv * n2 + j] = t;
      }
    __syncthreads();
    const double inv = 1.0 / W[(long long)k * n2 + k];
    __syncthreads();
    for (int j = threadIdx.x; j < n2; j += 256) W[(long long)k * n2 + j] *= inv;
    for (int i = threadIdx.x; i < r; i += 256) fac[i] = W[(long long)i * n2 + k];
    __syncthreads();
    for (long long t = threadIdx.x; t < (long long)r * n2; t += 256) {
      const int i = (int)(t / n2), j = (int)(t % n2);
      if (i != k) W[t] = fma(-fac[i], W[(long long)k * n2 + j], W[t]);
    }
    __syncthreads();
  }
  for (long long t = threadIdx.x; t < (long long)r * r; t += 256)
    Minv[(long long)b * r * r + t] = W[(t / r) * n2 + r + t % r];
}

__global__ void gather_dofs_kernel(long long n, int B, const int* __restrict__ ids, const double* __restrict__ field,
                                   long long fbs, long long n_nodes, double* __restrict__ out) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (q >= n) return;
  const long long dof = ids[q];
  out[(long long)b * n + q] = field[(long long)b * fbs + (dof % 3) * n_nodes + dof / 3];
}

}  // namespace

void launch_transfer(const XferMap& m, const double* src, long long cs, long long bs_src, double* dst,
                     long long bs_dst, int batch, const int* active, cudaStream_t s) {
  if (m.n == 0) return;
  launch_k(transfer_kernel, dim3(cdiv(3LL * m.n, 128), batch), dim3(128), 0, s, m.n, m.idx, m.xi, m.out, src, cs,
           bs_src, dst, bs_dst, active, 0);
  debug_check("transfer_kernel", s);
}

void launch_transfer_trace(const XferMap& m, const double* src, long long cs, long long bs_src, int slot, int batch,
                           const int* active, cudaStream_t s) {
  if (m.n == 0) return;
  const long long bs = 3LL * m.n;
  launch_k(transfer_kernel, dim3(dim3(cdiv(3LL * m.n, 128), batch)), dim3(128), 0, s, m.n, m.idx, m.xi, m.out, src, cs, bs_src,
                                                                      m.trace + (long long)slot * batch * bs, bs,
                                                                      active, 1);
  debug_check("transfer_kernel(trace)", s);
}

void launch_trace_interp(const XferMap& m, int lo, double alpha, double* dst, long long bs_dst, int batch,
                         const int* active, cudaStream_t s) {
  if (m.n == 0) return;
  launch_k(trace_interp_kernel, dim3(dim3(cdiv(m.n, 128), batch)), dim3(128), 0, s, m.n, m.out, m.trace, 3LL * m.n * batch, lo, alpha,
                                                                    dst, bs_dst, active);
  debug_check("trace_interp_kernel", s);
}

void launch_rom_minv(int r, int B, const double* Kbar, const double* e, double c, double* work, double* Minv,
                     cudaStream_t s) {
  rom_minv_kernel<<<B, 256, sizeof(double) * r, s>>>(r, Kbar, e, c, work, Minv);
  debug_check("rom_minv_kernel", s);
}

size_t rom_newton_smem(int r, int r_b, int nf) {
  return sizeof(double) * ((size_t)3 * r + r_b + nf + (size_t)r * (r + 1));
}

void launch_rom_newton(const RomLaunch& L, const double* ut, long long uts, const double* gsrc, long long gstride,
                       int gchunks, int n_slots, cudaStream_t s) {
  const size_t smem = rom_newton_smem(L.r, L.r_b, L.nf);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(rom_newton_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_k(rom_newton_kernel, dim3(L.B), dim3(256), smem, s, L, ut, uts, gsrc, gstride, gchunks, n_slots);
  debug_check("rom_newton_kernel", s);
}

void launch_rom_implicit(const RomLaunch& L, const double* ut, long long uts, int n_slots, cudaStream_t s) {
  launch_k(rom_implicit_kernel, dim3(L.B), dim3(256), sizeof(double) * L.r, s, L, ut, uts, n_slots);
  debug_check("rom_implicit_kernel", s);
}

void launch_step_begin(Ctl c, int B, cudaStream_t s) { launch_k(step_begin_kernel, dim3(1), dim3(256), 0, s, c, B); }

// The epilogues of a folded batched-ROM group and K3, one block per sample b: for every ROM in group order and
// every row (thread-strided), a^' = e_b sum_z part[z][i + r b] (splits in order), v^' = v^ + dt/2 (a^ + a^'),
// u^' = u~, and the norm terms; the block sums them in a fixed order and runs K3's test for b (finalize_kernel's
// body).  Frozen samples (converged, R29) keep their state.
constexpr int EF_T = 1024;
__global__ void __launch_bounds__(EF_T) rom_epi_finalize_kernel(const EpiArgs A, Ctl c) {
  pdl_enter();
  __shared__ double red[2][EF_T / 32];
  const int b = blockIdx.x, t = threadIdx.x;
  const int n = *c.n_dev + 1;
  const bool on = c.active[b] != 0;
  double num = 0.0, den = 0.0;
  if (on)
    for (int q = 0; q < A.n_sd; ++q) {
      const EpiSub& d = A.s[q];
      const long long col = (long long)d.r * b;
      for (int i = t; i < d.r; i += EF_T) {
        const long long id = col + i;
        const double* pp = d.part + id;
        const size_t zs = (size_t)d.r * A.B;
        double pv[16];  // the split partials in flight together (S <= 16 for these products), summed in order
#pragma unroll
        for (int z = 0; z < 16; ++z) pv[z] = z < d.S ? pp[z * zs] : 0.0;
        double araw = 0.0;
#pragma unroll
        for (int z = 0; z < 16; ++z)
          if (z < d.S) araw += pv[z];
        for (int z = 16; z < d.S; ++z) araw += pp[z * zs];
        const double an = d.e[b] * araw;
        const double un = d.Z[i + (long long)d.rz * b];
        const double vn = fma(0.5 * A.dt, d.ah0[id] + an, d.vh0[id]);
        if (A.with_norm) {
          const double dd = (un - d.uh1[id]) + A.dt * (vn - d.vh1[id]);
          const double w = un + A.dt * vn;
          num = fma(dd, dd, num);
          den = fma(w, w, den);
        }
        d.uh1[id] = un;
        d.vh1[id] = vn;
        d.ah1[id] = an;
      }
    }
  num = warp_sum(num);
  den = warp_sum(den);
  if ((t & 31) == 0) {
    red[0][t >> 5] = num;
    red[1][t >> 5] = den;
  }
  __syncthreads();
  if (t == 0) {
    num = 0.0;
    den = 0.0;
    for (int w = 0; w < EF_T / 32; ++w) {
      num += red[0][w];
      den += red[1][w];
    }
    if (on) {
      c.iters[b] = n;
      if (n >= A.min_iters) {
        c.numden[2 * b] = num;
        c.numden[2 * b + 1] = den;
        if (c.trace && n <= c.trace_T) {
          double* tr = c.trace + 2 * (((long long)(*c.step_dev - 1) * c.trace_T + (n - 1)) * A.B + b);
          tr[0] = num;
          tr[1] = den;
        }
        if (!isfinite(num) || !isfinite(den)) {
          c.flags[1] = 1;
          c.sticky[0] = 1;
        }
        bool conv = (num == 0.0) || (num < A.tol_rel * A.tol_rel * den);
        if (A.tol_abs > 0.0) conv = conv || (num < A.tol_abs * A.tol_abs);
        if (conv) c.active[b] = 0;
      }
    }
  }
}

int launch_rom_epi_finalize(const EpiArgs& A, Ctl c, cudaStream_t s) {
  launch_k(rom_epi_finalize_kernel, dim3(A.B), dim3(EF_T), 0, s, A, c);
  debug_check("rom_epi_finalize_kernel", s);
  launch_k(any_active_kernel, dim3(1), dim3(std::min(1024, (A.B + 31) / 32 * 32)), 0, s, c, A.B);
  debug_check("any_active_kernel", s);
  return 2;
}

int launch_finalize(Ctl c, const double2* partial, int n_slots, int B, int min_iters, double tol_rel,
                    double tol_abs, cudaStream_t s) {
  // B > 1: the controller update in a launch of its own (doing it in the last block to finish, through an arrival
  // counter, measured slower on c5: 10.24k vs 10.70k steps/s)
  // block size: enough warps for the slots (fewer idle warps per sample when there are few slots, e.g. c5)
  const int nt = std::min(FIN_T, std::max(32, (n_slots + 31) / 32 * 32));
  launch_k(finalize_kernel, dim3(B), dim3(nt), 0, s, c, partial, n_slots, B, min_iters, tol_rel, tol_abs,
           B == 1 ? 1 : 0);
  debug_check("finalize_kernel", s);
  if (B == 1) return 1;
  launch_k(any_active_kernel, dim3(1), dim3(std::min(1024, (B + 31) / 32 * 32)), 0, s, c, B);
  debug_check("any_active_kernel", s);
  return 2;
}

__global__ void rom_features_kernel(int nf, int B, const int* __restrict__ idx, const double* __restrict__ u,
                                    long long us, double* __restrict__ F, long long fs) {
  pdl_enter();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (q >= nf) return;
  const double* ub = u + us * b;
  const int i = idx[3 * q], j = idx[3 * q + 1], l = idx[3 * q + 2];
  double v = ub[i] * ub[j];
  if (l >= 0) v *= ub[l];
  F[q + fs * b] = v;
}

void launch_rom_features(int nf, int B, const int* idx, const double* u, long long us, double* F, long long fs,
                         cudaStream_t s) {
  if (nf == 0) return;
  launch_k(rom_features_kernel, dim3(dim3(cdiv(nf, 256), B)), dim3(256), 0, s, nf, B, idx, u, us, F, fs);
  debug_check("rom_features_kernel", s);
}

int rom_gchunks(long long n_s) { return (int)std::max<long long>(1, cdiv(n_s, GCHUNK)); }

int rom_partial_slots(int r, bool tc) { return (int)(tc ? cdiv(r, 256) : cdiv(r, 8)); }

// a^'[i] = e (sum_j KBF[i, j] z[j]) with z = [u~; x_d], x_d[t] = src[xd_idx[t]] (the FOM values the folded
// exchange reads), then rom_update_kernel's finish (v^', u^' = u~, norm partials).  B = 1.  One block per row:
// its 256 threads read the row and z with every load in flight at once (a warp-per-row loop is a chain of L2
// round trips), then a fixed-order block sum; the row is fixed at bind and read before the wait.  One norm
// partial slot per row (K3 sums the slots in order).
constexpr int FU_T = 256, FU_PER = 8;  // threads, row entries per thread held in registers (rows <= 2048)
__global__ void __launch_bounds__(FU_T) rom_fold_update_kernel(const RomLaunch L, const double* __restrict__ KBF,
                                                               const int* __restrict__ xd_idx, int n_xd,
                                                               const double* __restrict__ src) {
  pdl_launch();
  const int i = blockIdx.x, t = threadIdx.x;
  const int r = L.r, nz = L.r + n_xd;
  const double* row = KBF + (long long)i * nz;
  double k[FU_PER];
  int xi[FU_PER];
#pragma unroll
  for (int m = 0; m < FU_PER; ++m) {
    const int j = t + FU_T * m;
    k[m] = j < nz ? row[j] : 0.0;
    xi[m] = (j >= r && j < nz) ? xd_idx[j - r] : 0;
  }
  pdl_wait();
  double z[FU_PER];
#pragma unroll
  for (int m = 0; m < FU_PER; ++m) {
    const int j = t + FU_T * m;
    z[m] = j < r ? L.ustar[j] : (j < nz ? src[xi[m]] : 0.0);
  }
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < FU_PER; ++m) acc = fma(k[m], z[m], acc);
  for (int j = t + FU_T * FU_PER; j < nz; j += FU_T)  // rows longer than FU_T * FU_PER
    acc = fma(row[j], j < r ? L.ustar[j] : src[xd_idx[j - r]], acc);
  acc = block_sum256(acc);
  if (t == 0) {
    double num = 0.0, den = 0.0;
    if (L.active[0]) {
      const double an = L.e[0] * acc;
      const double vn = fma(0.5 * L.dt, L.ah0[i] + an, L.vh0[i]);
      const double un = L.ustar[i];
      if (L.with_norm) {
        const double d = (un - L.uh1[i]) + L.dt * (vn - L.vh1[i]);
        const double wv = un + L.dt * vn;
        num = d * d;
        den = wv * wv;
      }
      L.uh1[i] = un;
      L.vh1[i] = vn;
      L.ah1[i] = an;
    }
    L.partial[i] = make_double2(num, den);
  }
}

void launch_rom_fold_update(const RomLaunch& L, const double* KBF, const int* xd_idx, int n_xd, const double* src_field,
                            cudaStream_t s, int* launches) {
  launch_k(rom_fold_update_kernel, dim3(L.r), dim3(FU_T), 0, s, L, KBF, xd_idx, n_xd, src_field);
  debug_check("rom_fold_update_kernel", s);
  ++*launches;
}

void launch_rom_predict(const RomLaunch& L, cudaStream_t s, int* launches) {
  launch_k(rom_predict_kernel, dim3(cdiv((long long)L.r * L.B, 256)), dim3(256), 0, s, L.r, L.B, L.uh0, L.vh0, L.ah0, L.dt, L.c2,
           L.ustar);
  debug_check("rom_predict_kernel", s);
  ++*launches;
}

void launch_rom_advance(const RomLaunch& L, cudaStream_t s, int* launches) {
  if (L.r_b > 0)
    launch_k(rom_project_bnd_kernel, dim3(dim3(L.r_b, rom_gchunks(L.n_sdof), L.B)), dim3(256), 0, s, L.r_b, L.B, L.n_sdof, L.Phi_s,
                                                                                   L.s, L.gh);
  if (!L.pre)
    launch_k(rom_predict_kernel, dim3(cdiv((long long)L.r * L.B, 256)), dim3(256), 0, s, L.r, L.B, L.uh0, L.vh0, L.ah0,
             L.dt, L.c2, L.ustar);
  launch_rom_features(L.nf, L.B, L.feat_idx, L.ustar, L.r, L.F, L.nf, s);
  *launches += L.nf > 0;
  debug_check("rom_predict_kernel", s);
  if (L.beta > 0.0 && L.nf > 0) {  // implicit polynomial ROM: Newton (the features above are unused)
    launch_rom_newton(L, L.ustar, L.r, L.gh, 0, L.r_b > 0 ? L.gchunks : 0, rom_partial_slots(L.r, false), s);
    *launches += (L.r_b > 0) + 2;
    return;
  }
  launch_k(rom_update_kernel, dim3(dim3(cdiv(L.r, 8), L.B)), dim3(256), 0, s, L, L.beta > 0.0 ? 2 : 0);
  debug_check("rom_update_kernel", s);
  *launches += (L.r_b > 0) + (L.pre ? 1 : 2);
  if (L.beta > 0.0) {
    launch_rom_implicit(L, L.ustar, L.r, rom_partial_slots(L.r, false), s);
    ++*launches;
  }
}

void launch_rom_accel(const RomLaunch& L, const double* uh, double* ah, cudaStream_t s, int* launches) {
  RomLaunch A = L;
  A.ustar = const_cast<double*>(uh);
  A.ah1 = ah;
  launch_rom_features(L.nf, L.B, L.feat_idx, uh, L.r, L.F, L.nf, s);
  *launches += L.nf > 0;
  if (L.r_b > 0)
    launch_k(rom_project_bnd_kernel, dim3(dim3(L.r_b, rom_gchunks(L.n_sdof), L.B)), dim3(256), 0, s, L.r_b, L.B, L.n_sdof, L.Phi_s,
                                                                                   L.s, L.gh);
  launch_k(rom_update_kernel, dim3(dim3(cdiv(L.r, 8), L.B)), dim3(256), 0, s, A, 1);
  debug_check("rom_update_kernel", s);
  *launches += (L.r_b > 0) + 1;
}

void launch_rom_lift(int r, int B, long long nl, const double* Phi_lift, const int* code, const double* uh,
                     const double* sv, long long ns, double* out, cudaStream_t st) {
  if (nl == 0) return;
  launch_k(rom_lift_kernel, dim3(cdiv(cdiv(nl, LIFT_ROWS) * B * 32, 256)), dim3(256), 0, st, r, B, nl, Phi_lift, code, uh,
           sv, ns, out);
  debug_check("rom_lift_kernel", st);
}

cudaError_t launch_rom_project(long long nrows, int r, int B, const double* Phi, const int* ids, const double* field,
                               long long fbs, long long n_nodes, double* out, cudaStream_t s) {
  const int nz = (int)std::max<long long>(1, cdiv(nrows, PCHUNK));
  double* part = nullptr;
  const cudaError_t e = cudaMallocAsync((void**)&part, sizeof(double) * (size_t)nz * r * B, s);
  if (e != cudaSuccess) return e;
  rom_project_kernel<<<dim3(r, nz, B), 256, 0, s>>>(nrows, r, B, Phi, ids, field, fbs, n_nodes, part);
  debug_check("rom_project_kernel", s);
  sum_chunks_kernel<<<cdiv((long long)r * B, 256), 256, 0, s>>>(r, B, nz, part, out);
  return cudaFreeAsync(part, s);
}

void launch_gather_dofs(long long n, int B, const int* ids, const double* field, long long fbs, long long n_nodes,
                        double* out, cudaStream_t s) {
  if (n == 0) return;
  gather_dofs_kernel<<<dim3(cdiv(n, 256), B), 256, 0, s>>>(n, B, ids, field, fbs, n_nodes, out);
  debug_check("gather_dofs_kernel", s);
}

}  // namespace osam
