// K1: fused FOM advance -- explicit Newmark (beta = 0, gamma = 1/2) step of a hex8
// linear-elastic box subdomain with lumped mass (A.1 P:L1934-1947).
//
// State (R30): q = u + dt w (the next step's predictor) and w = v + dt/2 a, with the
// boundary values stored in q (0 on Dirichlet DOFs, the current Schwarz values s on Schwarz DOFs,
// written there by the transfer K2).  One launch computes, from the staged field X and the
// per-node field W:
//
//   f  = K X                   (matrix-free 27-point merged hex8 stencil, 153 nonzeros/node)
//   a  = -f / m_L ,  W' = W + cw a ,  Q' = X + cq W'      on free DOFs
//   W' = a = 0 ,  Q' = X                                   on constrained DOFs
//   partial sums  num = ||dt (W' - W'_prev)/2||^2 ,  den = ||X + dt (W + cv a)||^2   (free DOFs)
//
// A Schwarz sweep (X = q, W = w of the checkpoint; cw = cq = dt, cv = dt/2) is exactly
//   u* = u + dt v + dt^2/2 a (the Newmark predictor, = q),  a' = -K u*/m,
//   v' = v + dt/2 (a + a') = w + dt/2 a',  w' = w + dt a',  q' = u* + dt w',
// and the convergence change (u* - u*_prev) + dt (v' - v'_prev) = dt (w' - w'_prev)/2 on free DOFs
// because u* depends on the checkpoint only (eq:conv_criterion P:L443-467).  Other coefficient
// choices convert the state (initial condition: X = u0, W = v0, cw = dt/2; a new dt; v for output).
//
// One launch of the tiled kernel makes a K1 (kernels of their own: K1S, the gather path for small
// boxes; NL1 for the nonlinear materials; the excluded last x column's copy):
//   * its tile CTAs cover every node.  A block owns a TX x TY tile in (x, y) and a balanced
//     chunk of node planes in z.  One thread streams X planes (tile + halo) with 4D TMA loads into
//     a 4-deep ring guarded by full/empty mbarriers (no block-wide barrier in the loop: warps only
//     wait for data, the producer waits for the slowest warp to release a stage).  Each thread
//     forms, per staged plane and component, the 9 parity combinations of its 3x3 in-plane
//     neighbourhood and applies them to the forces of node planes m+1, m, m-1 held in registers
//     (2.5D streaming; the accumulator roles move through three register slots once per plane).
//     Two tile shapes are compiled from k1_tiled.cuh and picked per subdomain by k1_shape: 32 x 4 (a
//     warp is one x-row, so the (y, z) boundary class is warp-uniform) and 16 x 8 (a warp is two
//     16-node rows; for boxes whose x extent leaves most of a 32-wide column idle).  Interior rows use
//     the parity-reduced interior stencil, face rows their class table (out of line).  Lanes on an
//     x-face write it only when the face is fully constrained (no force needed).
//   * its extra CTAs (after the tile CTAs) gather the x-faces with free DOFs: 4 lanes per node, one
//     per z-offset, class table, fixed-order shuffle sum (xface_body).
// No atomics; every sum has a fixed order, so results are bitwise repeatable.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "osam_internal.h"

namespace cg = cooperative_groups;

namespace osam {

namespace {


__device__ __forceinline__ long long gidx(const Geom& g, int i, int j, int k) {
  return i + (long long)g.px * j + g.plane * k;
}

__device__ __forceinline__ int axis_class(int idx, int nn) { return idx == 0 ? 0 : (idx == nn - 1 ? 2 : 1); }

// free-DOF mask (bit c) of a node: Dirichlet > Schwarz > free (readings R12, R13)
__device__ __forceinline__ unsigned free_mask(const Geom& g, const Faces& F, int i, int j, int k) {
  unsigned dm = 0;
  bool sw = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const int v = ax == 0 ? i : (ax == 1 ? j : k);
    const bool on = v == ((f & 1) ? g.nn[ax] - 1 : 0);
    if (on) {
      dm |= F.dir[f];
      sw = sw || F.sw[f];
    }
  }
  return sw ? 0u : (~dm) & 7u;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Fixed-order block reduction of (num, den) -> partial[slot].
template <int N>
__device__ __forceinline__ void block_partial(double num, double den, double2* partial, int slot) {
  __shared__ double red[2][N / 32];
  const int t = threadIdx.x + blockDim.x * threadIdx.y;
  num = warp_sum(num);
  den = warp_sum(den);
  if ((t & 31) == 0) {
    red[0][t >> 5] = num;
    red[1][t >> 5] = den;
  }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int w = 0; w < N / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    partial[slot] = make_double2(a, b);
  }
}

// ---- TMA / mbarrier helpers (sm_90+ PTX; SASS UTMALDG + SYNCS) ----------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try(unsigned long long* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
#ifndef OSAM_BACKOFF
#define OSAM_BACKOFF 64  // ns between polls of a pending mbarrier phase (frees issue slots; measured +3.6%)
#endif
#if OSAM_BACKOFF > 0
  while (!mbar_try(bar, phase)) __nanosleep(OSAM_BACKOFF);
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
#ifdef OSAM_HINT
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, " OSAM_HINT ";\n"
#else
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
#endif
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
#endif
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int c,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(c), "r"(smem_u32(bar))
      : "memory");
}


inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// ---- K1 tiled kernel, one instance per tile shape (k1_tiled.cuh) --------------------------------
// k1a: 32 x OSAM_TY (default 4) -- a warp is one x-row; k1b: 16 x 8 -- a warp is two 16-node rows, for
// boxes whose x extent leaves most of a 32-wide tile column idle (c3: 142 / 111 nodes).  k1_shape picks
// per subdomain from the lane occupancy of the two tilings.
#ifndef OSAM_TY
#define OSAM_TY 4
#endif
#ifndef OSAM_ZC
#define OSAM_ZC 24  // target z-planes per CTA, 32 x TY tiles
#endif
#ifndef OSAM_ZC_B
#define OSAM_ZC_B 24  // the same, 16 x 8 tiles
#endif
namespace k1a {
#define K1_TX 32
#define K1_TY OSAM_TY
#define K1_ZC OSAM_ZC
#include "k1_tiled.cuh"
#undef K1_TX
#undef K1_TY
#undef K1_ZC
}  // namespace k1a
namespace k1b {
#define K1_TX 16
#define K1_TY 8
#define K1_ZC OSAM_ZC_B
#include "k1_tiled.cuh"
#undef K1_TX
#undef K1_TY
#undef K1_ZC
}  // namespace k1b
#ifndef OSAM_ZC_C
#define OSAM_ZC_C 24
#endif
namespace k1c {  // 48 x 2: three warps per tile, 5 CTAs per SM; long TMA rows (416-byte X, 384-byte W)
#define K1_TX 48
#define K1_TY 2
#define K1_ZC OSAM_ZC_C
#define K1_MINB 5
#include "k1_tiled.cuh"
#undef K1_TX
#undef K1_TY
#undef K1_ZC
}  // namespace k1c

// Tile shape of a subdomain's K1 (0: k1a, 1: k1b): the fraction of lanes that own a node, over x (the
// tile columns, the excluded last column not counted) and y; k1b only when it is clearly better (it
// pays ~1% in the two-row warps).  OSAM_K1_SHAPE=0/1 forces one.  Chosen once per subdomain by
// choose_fom_path (at create and at bind, with the TMA descriptors) and read from Faces::shape by every
// launch, so the shape, the descriptors and the partial-slot counts always agree.
static int k1_shape_choice(const Geom& g, const Faces& f) {
  const char* e = getenv("OSAM_K1_SHAPE");
  if (e && (e[0] == '0' || e[0] == '1' || e[0] == '2')) return e[0] - '0';
  auto occ = [&](int tx, int ty, int cols, bool xl) {
    const double nx = (double)(xl ? g.nn[0] - 1 : g.nn[0]);
    return nx / ((double)cols * tx) * (double)g.nn[1] / ((double)((g.nn[1] + ty - 1) / ty) * ty);
  };
  const double a = occ(k1a::TX, k1a::TY, k1a::tile_cols(g, f), k1a::xlast_excluded(g, f));
  const double b = occ(k1b::TX, k1b::TY, k1b::tile_cols(g, f), k1b::xlast_excluded(g, f));
  const double c = occ(k1c::TX, k1c::TY, k1c::tile_cols(g, f), k1c::xlast_excluded(g, f));
  // 48 x 2 for a box whose x extent it fits clearly better (opt-in: on c3's Omega1 the launch alone is 2.5% faster,
  // the concurrent step with Omega2's 16 x 8 CTAs 1.3% slower, profiles/r3_k1_experiments.md)
  static const bool use_c = getenv("OSAM_K1_C") && getenv("OSAM_K1_C")[0] == '1';
  if (use_c && c > 1.03 * a && c >= b) return 2;
  return b > 1.03 * a ? 1 : 0;
}
int k1_shape(const Geom&, const Faces& f) { return f.shape; }

#ifndef OSAM_NL_UNROLL
#define OSAM_NL_UNROLL 2
#endif
constexpr int NL_UNROLL = OSAM_NL_UNROLL;  // NL1: unroll of the Gauss-point loop


// Small subdomains (K1S): the TMA-streamed tiled kernel pays a load round trip per z-plane inside each
// CTA, which dominates for boxes of a few thousand nodes (c1, c2).  Here every node gathers its three planes
// at once (class-table stencil) from the L2-resident field.
// Groups of 32 nodes, 3 warps each: warp 3 g + o gathers the plane oz = o - 1 for group g's 32 nodes, so the lanes
// of a warp read the same coefficient offsets (one class-table address per load for a warp of interior nodes
// instead of up to 24 with 4 lanes per node); the three plane contributions meet in shared memory and the group's
// first warp sums them in the order (oz = -1 + oz = 0) + oz = +1 -- every force component is the same FMA chain as
// with 4 lanes per node, bitwise (and as small_resident_kernel's).  2 groups = 64 nodes per block (measured: c2 18.3k /
// 21.2k / 19.6k steps/s with 1 / 2 / 4 groups; the persistent small controller 11.1k / 17.4k / 19.4k).
constexpr int GGRP = 2;
constexpr int GB = 96 * GGRP;
constexpr int GNODES = 32 * GGRP;
__device__ __forceinline__ void gather_body(const FomLaunch& L, int blk) {
  __shared__ double sf[GGRP][3][3][32];
  const Geom& g = L.g;
  const long long np = g.npad;
  const long long n = (long long)g.nn[0] * g.nn[1] * g.nn[2];
  const int lane = threadIdx.x & 31, wz = threadIdx.x >> 5;
  const int grp = wz / 3, o = wz % 3;
  const long long t = (long long)blk * GNODES + grp * 32 + lane;
  const bool valid = t < n;
  const int i = valid ? (int)(t % g.nn[0]) : 0;
  const int j = valid ? (int)((t / g.nn[0]) % g.nn[1]) : 0;
  const int k = valid ? (int)(t / ((long long)g.nn[0] * g.nn[1])) : 0;
  const int cx = axis_class(i, g.nn[0]), cy = axis_class(j, g.nn[1]), cz = axis_class(k, g.nn[2]);
  double f[3] = {0.0, 0.0, 0.0};
  const int oz = o - 1;
  if (valid && k + oz >= 0 && k + oz <= g.nn[2] - 1) {
    const double* coef = L.coef + (size_t)(cx + 3 * (cy + 3 * cz)) * 27 * 9;
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy) {
      if (j + oy < 0 || j + oy > g.nn[1] - 1) continue;
#pragma unroll
      for (int ox = -1; ox <= 1; ++ox) {
        if (i + ox < 0 || i + ox > g.nn[0] - 1) continue;
        const long long q = gidx(g, i + ox, j + oy, k + oz);
        const double x[3] = {__ldg(L.x + q), __ldg(L.x + np + q), __ldg(L.x + 2 * np + q)};
        const double* cb = coef + ((ox + 1) + 3 * ((oy + 1) + 3 * (oz + 1))) * 9;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) f[c] = fma(__ldg(cb + c * 3 + d), x[d], f[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) sf[grp][o][c][lane] = f[c];
  __syncthreads();
  if (o == 0)
#pragma unroll
    for (int c = 0; c < 3; ++c) f[c] = (sf[grp][0][c][lane] + sf[grp][1][c][lane]) + sf[grp][2][c][lane];
  const int sub = o;  // the group's first warp finishes its nodes
  double num = 0.0, den = 0.0;
  if (valid && sub == 0) {
    const long long id = gidx(g, i, j, k);
    const unsigned fm = free_mask(g, L.f, i, j, k);
    const double inv_m = L.inv_mass[(cx == 1 ? 1 : 0) + (cy == 1 ? 2 : 0) + (cz == 1 ? 4 : 0)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = __ldg(L.x + c * np + id);
      double an = 0.0, wn = 0.0, qn = x;
      if ((fm >> c) & 1) {
        const double w0 = L.w0[c * np + id];
        an = -f[c] * inv_m;
        wn = fma(L.cw, an, w0);
        qn = fma(L.cq, wn, x);
        const double w = fma(L.dt, fma(L.cv, an, w0), x);
        if (L.with_norm) {
          const double d = L.z_out ? w - L.z_out[c * np + id] : 0.5 * L.dt * (wn - L.w_out[c * np + id]);
          num = fma(d, d, num);
          den = fma(w, w, den);
        }
        if (L.z_out) L.z_out[c * np + id] = w;
      }
      if (L.q_out) L.q_out[c * np + id] = qn;
      L.w_out[c * np + id] = wn;
      if (L.a_out) L.a_out[c * np + id] = an;
    }
  }
  block_partial<GB>(num, den, L.partial, blk);
}

__global__ void __launch_bounds__(GB) fom_gather_kernel(const FomLaunch L) {
  pdl_enter();
  gather_body(L, blockIdx.x);
}

// ---- persistent controller for small all-FOM groups (see osam_internal.h SmallArgs) ---------------
__device__ __forceinline__ void small_xfer(const SmallArgs& A, int i, int mi, bool first, int k) {
  auto cb = [&](int j) { return (k & 1) ? 1 - A.s[j].cur0 : A.s[j].cur0; };
  const SmallSub& d = A.s[i];
  const SmallMap& m = d.maps[mi];
  const SmallSub& src = A.s[m.src];
  const bool newest = (m.src < i) || !first;  // iterate n of an earlier source, else n - 1 (n = 1: checkpoint u)
  const double* field = src.st[newest ? cb(m.src) : 1 - cb(m.src)][0];
  double* dstq = d.st[cb(i)][0];
  const long long cs = src.L.g.npad;
  for (long long t = blockIdx.x * (long long)GB + threadIdx.x; t < 3LL * m.n; t += (long long)gridDim.x * GB) {
    const int p = (int)(t / 3), cc = (int)(t - 3LL * p);
    const int o = m.out[3 * p + cc];
    if (o < 0) continue;
    const double xx = m.xi[3 * p], yy = m.xi[3 * p + 1], zz = m.xi[3 * p + 2];
    const double* sb = field + cc * cs;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double w = ((q & 1) ? xx : 1.0 - xx) * ((q & 2) ? yy : 1.0 - yy) * ((q & 4) ? zz : 1.0 - zz);
      acc = fma(w, sb[m.idx[8 * p + q]], acc);
    }
    dstq[o] = acc;
  }
}

__device__ __forceinline__ void small_step_begin(const Ctl& C) {
  C.active[0] = 1;
  C.iters[0] = 0;
  C.flags[0] = 1;
  C.flags[1] = 0;
  *C.n_dev = 0;
  *C.step_dev += 1;
}

// CLUSTER: the whole group runs as one thread-block cluster (<= 16 CTAs, each looping over its node blocks)
// and the phases are separated by cluster barriers (barrier.cluster arrive.release / wait.acquire: global
// writes of the phase are visible after it) instead of grid-wide cooperative barriers
template <bool CLUSTER>
__device__ __forceinline__ void phase_sync() {
  if (CLUSTER)
    cg::this_cluster().sync();
  else
    cg::this_grid().sync();
}

template <bool CLUSTER>
__global__ void __launch_bounds__(GB) small_persistent_kernel(const __grid_constant__ SmallArgs A) {
  __shared__ double red[2][GB / 32];
  const Ctl& C = A.ctl;
  int total_vb = 0;
  for (int i = 0; i < A.n_sd; ++i) total_vb += A.s[i].nvb;
  if (blockIdx.x == 0 && threadIdx.x == 0) small_step_begin(C);  // later steps begin inside K3 below
  phase_sync<CLUSTER>();
  for (int k = 0; k < A.n_steps; ++k) {
    auto cb = [&](int i) { return (k & 1) ? 1 - A.s[i].cur0 : A.s[i].cur0; };
    for (int n = 1; n <= A.max_iters; ++n) {
      const bool first = n == 1;
      // K2 in sweep order, one phase per destination (a single phase for all of them, where no transfer
      // reads another destination's output, measured slower on c1: 13.9k vs 18.3k steps/s)
      for (int i = 0; i < A.n_sd; ++i) {
        for (int mi = 0; mi < A.s[i].n_maps; ++mi) small_xfer(A, i, mi, first, k);
        if (A.s[i].n_maps) phase_sync<CLUSTER>();
      }
      // K1S of every subdomain (no transfer reads a FOM advance's output, R30)
      for (int vb = blockIdx.x; vb < total_vb; vb += gridDim.x) {
        int i = 0, b = vb;
        while (b >= A.s[i].nvb) b -= A.s[i++].nvb;
        const SmallSub& d = A.s[i];
        const int c = cb(i), x = 1 - c;
        FomLaunch L = d.L;
        L.x = d.st[c][0];
        L.w0 = d.st[c][1];
        L.q_out = d.st[x][0];
        L.w_out = d.st[x][1];
        L.with_norm = first ? 0 : 1;
        L.partial = A.partial + d.slot0;
        gather_body(L, b);
        __syncthreads();  // block_partial's scratch is reused by the next node block
      }
      phase_sync<CLUSTER>();
      // K3 and the controller flags (block 0; fixed-order sums); the continue decision goes through A.go so
      // that the next step's begin can be written here too
      if (blockIdx.x == 0) {
        double num = 0.0, den = 0.0;
        if (n >= A.min_iters)
          for (int sl = threadIdx.x; sl < A.n_slots; sl += GB) {
            num += A.partial[sl].x;
            den += A.partial[sl].y;
          }
        num = warp_sum(num);
        den = warp_sum(den);
        if ((threadIdx.x & 31) == 0) {
          red[0][threadIdx.x >> 5] = num;
          red[1][threadIdx.x >> 5] = den;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          num = den = 0.0;
          for (int w = 0; w < GB / 32; ++w) {
            num += red[0][w];
            den += red[1][w];
          }
          if (C.active[0]) {
            C.iters[0] = n;
            if (n >= A.min_iters) {
              C.numden[0] = num;
              C.numden[1] = den;
              if (C.trace && n <= C.trace_T) {  // convergence trace (osam_set_conv_trace), B = 1
                double* tr = C.trace + 2 * ((long long)(*C.step_dev - 1) * C.trace_T + (n - 1));
                tr[0] = num;
                tr[1] = den;
              }
              if (!isfinite(num) || !isfinite(den)) {
                C.flags[1] = 1;
                C.sticky[0] = 1;
              }
              bool conv = (num == 0.0) || (num < A.tol_rel * A.tol_rel * den);
              if (A.tol_abs > 0.0) conv = conv || (num < A.tol_abs * A.tol_abs);
              if (conv) C.active[0] = 0;
            }
          }
          *C.n_dev = n;
          C.flags[0] = C.active[0];
          if (C.iters_all) C.iters_all[*C.step_dev - 1] = C.iters[0];
          if (C.active[0] && n >= A.max_iters) C.sticky[1] = 1;
          const int go = C.flags[0] && !C.flags[1] && n < A.max_iters;
          *A.go = go;
          if (!go && k + 1 < A.n_steps) small_step_begin(C);
        }
      }
      phase_sync<CLUSTER>();
      if (!*(volatile int*)A.go) break;
    }
  }
}

bool small_fom(const Geom& g) { return g.small != 0; }

void choose_fom_path_impl(Geom& g, Faces& f) {
  const char* e = getenv("OSAM_GATHER_MAX");
  const long long cap = e ? atoll(e) : (1LL << 18);
  g.small = (long long)g.nn[0] * g.nn[1] * g.nn[2] <= cap ? 1 : 0;
  f.shape = (unsigned char)k1_shape_choice(g, f);
}

__device__ __forceinline__ void surface_node(const Geom& g, long long t, int* i, int* j, int* k) {
  const long long n0 = g.nn[0], n1 = g.nn[1], n2 = g.nn[2];
  const long long sz = n0 * n1;
  if (t < 2 * sz) {
    const long long r = t % sz;
    *i = (int)(r % n0);
    *j = (int)(r / n0);
    *k = t < sz ? 0 : (int)(n2 - 1);
    return;
  }
  t -= 2 * sz;
  const long long sy = n0 * (n2 - 2);
  if (t < 2 * sy) {
    const long long r = t % sy;
    *i = (int)(r % n0);
    *k = 1 + (int)(r / n0);
    *j = t < sy ? 0 : (int)(n1 - 1);
    return;
  }
  t -= 2 * sy;
  const long long sx = (n1 - 2) * (n2 - 2);
  const long long r = t % sx;
  *j = 1 + (int)(r % (n1 - 2));
  *k = 1 + (int)(r / (n1 - 2));
  *i = t < sx ? 0 : (int)(n0 - 1);
}

__host__ __device__ inline long long surface_count(const Geom& g) {
  const long long n0 = g.nn[0], n1 = g.nn[1], n2 = g.nn[2];
  const long long inner = (n2 > 2 ? n2 - 2 : 0);
  return 2 * n0 * n1 + 2 * n0 * inner + 2 * (n1 > 2 ? n1 - 2 : 0) * inner;
}

__global__ void pack_kernel(Geom g, const double* __restrict__ src, double* __restrict__ dst, long long n) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const long long i = p % g.nn[0], j = (p / g.nn[0]) % g.nn[1], k = p / ((long long)g.nn[0] * g.nn[1]);
  const long long q = i + g.px * j + g.plane * k;
  for (int c = 0; c < 3; ++c) dst[c * g.npad + q] = src[c * n + p];
}

__global__ void unpack_kernel(Geom g, const double* __restrict__ src, double* __restrict__ dst, long long n) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const long long i = p % g.nn[0], j = (p / g.nn[0]) % g.nn[1], k = p / ((long long)g.nn[0] * g.nn[1]);
  const long long q = i + g.px * j + g.plane * k;
  for (int c = 0; c < 3; ++c) dst[c * n + p] = src[c * g.npad + q];
}

// Dirichlet u := 0, constrained w := 0 on every surface node (initial condition).
__global__ void zero_constrained_kernel(Geom g, Faces F, double* u, double* w) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= surface_count(g)) return;
  int i, j, k;
  surface_node(g, t, &i, &j, &k);
  const long long q = gidx(g, i, j, k);
  unsigned dm = 0;
  bool sw = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const int v = ax == 0 ? i : (ax == 1 ? j : k);
    if (v == ((f & 1) ? g.nn[ax] - 1 : 0)) {
      dm |= F.dir[f];
      sw = sw || F.sw[f];
    }
  }
  for (int c = 0; c < 3; ++c) {
    const bool dir = (dm >> c) & 1;
    if (dir || sw) w[c * g.npad + q] = 0.0;
    if (dir) u[c * g.npad + q] = 0.0;
  }
}



// the excluded x+ column (see xlast_excluded): Q' = X, W' = 0, a = 0 on every node of the face
// The excluded last x column: Q' = X (prescribed), W' = a = 0.  XL_PER nodes per thread with every
// load issued first (each node is its own cache line, so the kernel is latency-bound).
constexpr int XL_PER = 8;
__global__ void __launch_bounds__(128) xlast_copy_kernel(const FomLaunch L) {
  const Geom& g = L.g;
  const long long n = (long long)g.nn[1] * g.nn[2], np = g.npad;
  long long ids[XL_PER];
  double v[XL_PER][3];
#pragma unroll
  for (int q = 0; q < XL_PER; ++q) {
    const long long t = ((long long)blockIdx.x * XL_PER + q) * 128 + threadIdx.x;
    ids[q] = t < n ? gidx(g, g.nn[0] - 1, (int)(t % g.nn[1]), (int)(t / g.nn[1])) : -1;
#pragma unroll
    for (int c = 0; c < 3; ++c) v[q][c] = (ids[q] >= 0 && L.q_out) ? L.x[c * np + ids[q]] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < XL_PER; ++q) {
    if (ids[q] < 0) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (L.q_out) L.q_out[c * np + ids[q]] = v[q][c];
      L.w_out[c * np + ids[q]] = 0.0;
      if (L.a_out) L.a_out[c * np + ids[q]] = 0.0;
    }
  }
}






// ---- NL1: nonlinear FOM advance (SVK / Neohookean; App. A.2, A.3) ----------
// The explicit scheme and the (q, w) state of R30 are unchanged; only the internal force is the
// nonlinear weak form  f_a = sum_e sum_q detJ P(F_q) dN_a/dX(q),  F = I + grad u,  2x2x2 Gauss.
// A CTA owns a 16 x 14 node tile and a z-chunk of node planes, streams node planes through a 2-plane
// shared ring (18 x 16 staged nodes: the tile plus a 1-node halo), computes each element layer once
// per tile -- one thread per element (17 x 15 = 255 elements), 24 nodal force contributions into
// shared memory -- and finishes a node plane by gathering its 8 element contributions in a fixed
// order (deterministic; no atomics), then exactly K1's finish (a, w', q', norm partials).  256
// threads: the element code keeps 36 force accumulators plus a Gauss point's F, P in registers
// (no spills at <= 255 registers).
namespace nl {
constexpr int TXN = 16, TYN = 14, ZCN = 32;
// First node plane of z-chunk b of tz: the chunk sizes taper over the chunk layers (dispatched in order, bz slowest)
// from (1 + p/100) to (1 - p/100) of the mean, so the launch drains through short CTAs (as K1's zsplit, k1_tiled.cuh)
#ifndef OSAM_NL_ZTAPER
#define OSAM_NL_ZTAPER 60  // measured (profiles/r8d_ab_nl_ztaper.log): SVK 154.6 -> 159.2, Neohookean 106.0 -> 109.0 steps/s on c3
#endif
__device__ __forceinline__ int nl_zsplit(int nz, int tz, int b) {
  constexpr long long p = OSAM_NL_ZTAPER;
  if (p == 0 || tz < 2) return (int)((long long)b * nz / tz);
  const long long c = (long long)b * (100 + p) * (tz - 1) - p * (long long)b * (b - 1);
  return (int)((long long)nz * c / (100LL * tz * (tz - 1)));
}
constexpr int EX = TXN + 1, EY = TYN + 1, NE = EX * EY;
constexpr int PXN = TXN + 2, PYN = TYN + 2, PLN = PXN * PYN;
constexpr int NTN = 256;
constexpr int NN = TXN * TYN;  // nodes finished per plane
// X ring of 3 planes | element forces of 2 layers | W and W'_prev (or z_prev) of 2 node planes
constexpr size_t SMEM = sizeof(double) * (3 * 3 * PLN + 2 * 24 * NE + 2 * 2 * 3 * NN + 8 * 2 * 12);
}  // namespace nl

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int MAT>
__device__ __forceinline__ void pk1(const FomLaunch& L, const double F[3][3], double P[3][3]) {
  double C[3][3];  // symmetric: 6 products
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      C[i][j] = fma(F[0][i], F[0][j], fma(F[1][i], F[1][j], F[2][i] * F[2][j]));
      C[j][i] = C[i][j];
    }
  double S[3][3];
  if (MAT == OSAM_SVK) {  // S = lambda tr(E) I + 2 mu E, E = (C - I)/2
    const double trE = 0.5 * ((C[0][0] - 1.0) + (C[1][1] - 1.0) + (C[2][2] - 1.0));
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j) {
        S[i][j] = i == j ? fma(L.mat_mu, C[i][j] - 1.0, L.mat_lam * trE) : L.mat_mu * C[i][j];
        S[j][i] = S[i][j];
      }
  } else {  // Neohookean: S = kappa/2 (det C - 1) C^-1 + mu (det C)^(-1/3) (I - tr(C)/3 C^-1)
    const double a00 = C[1][1] * C[2][2] - C[1][2] * C[2][1], a01 = C[0][2] * C[2][1] - C[0][1] * C[2][2],
                 a02 = C[0][1] * C[1][2] - C[0][2] * C[1][1];
    const double det = C[0][0] * a00 + C[1][0] * a01 + C[2][0] * a02;
    const double id = 1.0 / det;
    double Ci[3][3];
    Ci[0][0] = a00 * id;
    Ci[0][1] = a01 * id;
    Ci[0][2] = a02 * id;
    Ci[1][0] = (C[1][2] * C[2][0] - C[1][0] * C[2][2]) * id;
    Ci[1][1] = (C[0][0] * C[2][2] - C[0][2] * C[2][0]) * id;
    Ci[1][2] = (C[0][2] * C[1][0] - C[0][0] * C[1][2]) * id;
    Ci[2][0] = (C[1][0] * C[2][1] - C[1][1] * C[2][0]) * id;
    Ci[2][1] = (C[0][1] * C[2][0] - C[0][0] * C[2][1]) * id;
    Ci[2][2] = (C[0][0] * C[1][1] - C[0][1] * C[1][0]) * id;
    const double sv = 0.5 * L.mat_kappa * (det - 1.0);
    const double sd = L.mat_mu * rcbrt(det);
    const double t3 = (C[0][0] + C[1][1] + C[2][2]) / 3.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) S[i][j] = sv * Ci[i][j] + sd * ((i == j ? 1.0 : 0.0) - t3 * Ci[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) P[i][j] = fma(F[i][0], S[0][j], fma(F[i][1], S[1][j], F[i][2] * S[2][j]));
}

// 24 nodal force contributions f[a][c] of one hex8 element (local node a = dx + 2 dy + 4 dz),
// rectangular, J = diag(h/2).  With N_a = prod_d (1 + s_ad xi_d)/2, dN_a/dX_j = s_aj/h_j prod_{d != j}
// w(a_d, q_d), w = (1 +- 1/sqrt3)/2 on the same / opposite side, so at Gauss point q
//     du_i/dX_j = sum_p W_j[p] (u_i(a_j = 1, p) - u_i(a_j = 0, p))    (p: the other two bits of a)
//     f_a,i     = sum_j s_aj T_j[i][p(a)],   T_j[i][p] = sum_q detJ P_q[i][j] W_j[p](q).
// The nodal displacements are read from the staged planes (u(a) = ua(a, c)); 36 accumulators T.
// The weights of point q, axis j, pair p (gradient: w w / h_j; accumulation: w w detJ / h_j) come from a
// per-CTA shared table wtab[q][0|1][j][p] (element_weights), read as broadcasts.
__device__ __forceinline__ void element_weights(const FomLaunch& L, double* wtab) {
  const double r3 = 0.57735026918962576451;  // 1/sqrt(3)
  const double gpl = 0.5 * (1.0 + r3), gmi = 0.5 * (1.0 - r3);
  const double detJ = 0.125 * L.g.h[0] * L.g.h[1] * L.g.h[2];
  for (int t = threadIdx.x; t < 8 * 2 * 12; t += blockDim.x) {
    const int q = t / 24, kind = (t / 12) % 2, j = (t % 12) / 4, p = t % 4;
    const int o1 = j == 0 ? 1 : 0, o2 = j == 2 ? 1 : 2;
    const double w1 = ((p & 1) == ((q >> o1) & 1)) ? gpl : gmi;
    const double w2 = (((p >> 1) & 1) == ((q >> o2) & 1)) ? gpl : gmi;
    const double wg = w1 * w2 * (1.0 / L.g.h[j]);
    wtab[t] = kind ? wg * detJ : wg;
  }
}

template <int MAT, class UA>
__device__ __forceinline__ void element_forces(const FomLaunch& L, UA ua, const double* __restrict__ wtab,
                                               double (&f)[8][3]) {
  double T[3][3][4], D[3][3][4];  // accumulators; edge differences u_i(a_j = 1, p) - u_i(a_j = 0, p)
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int o1 = j == 0 ? 1 : 0, o2 = j == 2 ? 1 : 2;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int a0 = ((p & 1) << o1) | (((p >> 1) & 1) << o2);
        T[j][i][p] = 0.0;
        D[j][i][p] = ua(a0 | (1 << j), i) - ua(a0, i);
      }
  }
#pragma unroll NL_UNROLL
  for (int q = 0; q < 8; ++q) {
    const double* wg = wtab + q * 24;  // [j][p] gradient weights, then [j][p] accumulation weights
    double F[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double gsum = 0.0;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          gsum = fma(wg[j * 4 + p], D[j][i][p], gsum);
        }
        F[i][j] = (i == j ? 1.0 : 0.0) + gsum;
      }
    }
    double P[3][3];
    pk1<MAT>(L, F, P);
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double wt = wg[12 + j * 4 + p];
#pragma unroll
        for (int i = 0; i < 3; ++i) T[j][i][p] = fma(P[i][j], wt, T[j][i][p]);
      }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int o1 = j == 0 ? 1 : 0, o2 = j == 2 ? 1 : 2;
        const int p = ((a >> o1) & 1) | (((a >> o2) & 1) << 1);
        v = ((a >> j) & 1) ? v + T[j][i][p] : v - T[j][i][p];
      }
      f[a][i] = v;
    }
}

template <int MAT>
__global__ void __launch_bounds__(nl::NTN, 1) fom_nl_kernel(const __grid_constant__ FomLaunch L) {
  using namespace nl;
  extern __shared__ __align__(16) double nsm[];
  double* Xs = nsm;                         // [3][3][PYN][PXN]   node planes, slot p mod 3
  double* EF = Xs + 3 * 3 * PLN;            // [2][8][3][NE]      element forces, layer mod 2
  double* Ws = EF + 2 * 24 * NE;            // [2][2][3][NN]      W, W'_prev (or z_prev), plane mod 2
  double* Wq = Ws + 2 * 2 * 3 * NN;         // [8][2][3][4]       Gauss weights (element_weights)
  const Geom& g = L.g;
  const long long np = g.npad;
  const int tid = threadIdx.x, tx = tid % TXN, ty = tid / TXN;
  const int ntx = (g.nn[0] + TXN - 1) / TXN, nty = (g.nn[1] + TYN - 1) / TYN;
  const int nzc = (g.nn[2] + ZCN - 1) / ZCN;
  const int bx = blockIdx.x % ntx, by = (blockIdx.x / ntx) % nty, bz = blockIdx.x / (ntx * nty);
  const int x0 = bx * TXN, y0 = by * TYN;
  const int kbeg = nl_zsplit(g.nn[2], nzc, bz), kend = nl_zsplit(g.nn[2], nzc, bz + 1) - 1;
  const int nelx = g.nn[0] - 1, nely = g.nn[1] - 1, nelz = g.nn[2] - 1;
  const bool need_prev = L.with_norm != 0;
  const double* prev = L.z_out ? L.z_out : L.w_out;  // previous iterate for the norm (read before written)

  // asynchronous copies (cp.async, zero-filled outside the box): node plane p, and W / previous for
  // the tile's nodes of plane p
  auto issue_plane = [&](int p) {
    double* dst = Xs + ((p + 3) % 3) * 3 * PLN;
    for (int t = tid; t < 3 * PLN; t += NTN) {
      const int c = t / PLN, rem = t % PLN, yy = rem / PXN, xx = rem % PXN;
      const int i = x0 - 1 + xx, j = y0 - 1 + yy;
      const bool ok = i >= 0 && i < g.nn[0] && j >= 0 && j < g.nn[1] && p >= 0 && p < g.nn[2];
      cp_async8(dst + t, ok ? L.x + c * np + gidx(g, i, j, p) : L.x, ok);
    }
  };
  auto issue_w = [&](int p) {
    if (p > kend) return;
    double* dst = Ws + (p & 1) * 2 * 3 * NN;
    const int i = x0 + tx, j = y0 + ty;
    if (ty < TYN && i < g.nn[0] && j < g.nn[1]) {
      const long long id = gidx(g, i, j, p);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cp_async8(dst + c * NN + tid, L.w0 + c * np + id, true);
        if (need_prev) cp_async8(dst + (3 + c) * NN + tid, prev + c * np + id, true);
      }
    }
  };
  auto compute_layer = [&](int l) {
    if (tid >= NE) return;
    const int lx = tid % EX, ly = tid / EX;
    const int ex = x0 - 1 + lx, ey = y0 - 1 + ly;
    double* out = EF + (l & 1) * 24 * NE + tid;
    if (ex < 0 || ex >= nelx || ey < 0 || ey >= nely || l < 0 || l >= nelz) {
#pragma unroll
      for (int q = 0; q < 24; ++q) out[q * NE] = 0.0;
      return;
    }
    const double* p0 = Xs + ((l + 3) % 3) * 3 * PLN + ly * PXN + lx;
    const double* p1 = Xs + ((l + 4) % 3) * 3 * PLN + ly * PXN + lx;
    auto ua = [&](int a, int c) { return ((a >> 2) ? p1 : p0)[c * PLN + ((a >> 1) & 1) * PXN + (a & 1)]; };
    double f[8][3];
    element_forces<MAT>(L, ua, Wq, f);
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) out[(a * 3 + c) * NE] = f[a][c];
  };

  double num = 0.0, den = 0.0;
  element_weights(L, Wq);  // visible after the prologue's barrier
  // prologue: planes kbeg-1, kbeg, kbeg+1 and W of plane kbeg; element layer kbeg-1
  issue_plane(kbeg - 1);
  issue_plane(kbeg);
  issue_plane(kbeg + 1);
  issue_w(kbeg);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  compute_layer(kbeg - 1);
  for (int k = kbeg; k <= kend; ++k) {
    __syncthreads();  // resident: planes k, k+1 and W(k); free: the slot of plane k-1 and W(k-1)
    issue_plane(k + 2);
    issue_w(k + 1);
    cp_async_commit();
    compute_layer(k);  // overlaps the copies
    __syncthreads();
    const int i = x0 + tx, j = y0 + ty;
    if (ty < TYN && i < g.nn[0] && j < g.nn[1]) {
      double fsum[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int dz = 0; dz < 2; ++dz)
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) {
            const int a = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
            const double* e = EF + ((k - 1 + dz) & 1) * 24 * NE + (tx + dx) + EX * (ty + dy);
#pragma unroll
            for (int c = 0; c < 3; ++c) fsum[c] += e[(a * 3 + c) * NE];
          }
      const long long id = gidx(g, i, j, k);
      const unsigned fm = free_mask(g, L.f, i, j, k);
      const double inv_m = L.inv_mass[(axis_class(i, g.nn[0]) == 1) + 2 * (axis_class(j, g.nn[1]) == 1) +
                                      4 * (axis_class(k, g.nn[2]) == 1)];
      const double* xo = Xs + (k % 3) * 3 * PLN + (ty + 1) * PXN + tx + 1;
      const double* wv = Ws + (k & 1) * 2 * 3 * NN + tid;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double x = xo[c * PLN];
        double an = 0.0, wn = 0.0, qn = x;
        if ((fm >> c) & 1) {
          const double w0 = wv[c * NN];
          an = -fsum[c] * inv_m;
          wn = fma(L.cw, an, w0);
          qn = fma(L.cq, wn, x);
          const double w = fma(L.dt, fma(L.cv, an, w0), x);
          if (need_prev) {
            const double pv = wv[(3 + c) * NN];
            const double d = L.z_out ? w - pv : 0.5 * L.dt * (wn - pv);
            num = fma(d, d, num);
            den = fma(w, w, den);
          }
          if (L.z_out) L.z_out[c * np + id] = w;
        }
        if (L.q_out) L.q_out[c * np + id] = qn;
        L.w_out[c * np + id] = wn;
        if (L.a_out) L.a_out[c * np + id] = an;
      }
    }
    cp_async_wait_all();
  }
  block_partial<nl::NTN>(num, den, L.partial, blockIdx.x);
}

int nl_ctas(const Geom& g) {
  using namespace nl;
  return ((g.nn[0] + TXN - 1) / TXN) * ((g.nn[1] + TYN - 1) / TYN) * ((g.nn[2] + ZCN - 1) / ZCN);
}

}  // namespace

int fom_partial_slots(const Geom& g, const Faces& f) {
  if (small_fom(g)) return (int)cdiv((long long)g.nn[0] * g.nn[1] * g.nn[2], GNODES);
  switch (k1_shape(g, f)) {
    case 1: return k1b::partial_slots(g, f);
    case 2: return k1c::partial_slots(g, f);
    default: return k1a::partial_slots(g, f);
  }
}

int fom_nl_partial_slots(const Geom& g) { return nl_ctas(g); }

bool fom_ingrid_xfer_ok(const Geom& g, const Faces& f, int material) {
  if (material != OSAM_LINEAR || small_fom(g) || g.nn[0] < 4) return false;
  for (int q = 2; q < 6; ++q)
    if (f.sw[q]) return false;
  return f.sw[0] || f.sw[1];
}

bool fom_small(const Geom& g) { return small_fom(g); }
void choose_fom_path(Geom& g, Faces& f) { choose_fom_path_impl(g, f); }

int small_persistent_grid() {
  static int g = 0;
  if (g == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_persistent_kernel<false>, GB, 0);
    g = std::max(1, sms * std::max(1, per_sm));
  }
  return g;
}

// One thread-block cluster of up to 16 CTAs (non-portable size; cluster barriers between the phases) when the
// group is small enough that its node blocks fit a few per CTA (OSAM_SMALL_CLUSTER=0: the grid-wide
// cooperative launch); otherwise every co-resident CTA with grid-wide barriers.
cudaError_t launch_small_persistent(const SmallArgs& A, cudaStream_t s) {
  int total_vb = 0;
  for (int i = 0; i < A.n_sd; ++i) total_vb += A.s[i].nvb;
  const bool cl_env = !(getenv("OSAM_SMALL_CLUSTER") && getenv("OSAM_SMALL_CLUSTER")[0] == '0');
  static int cl_max = -1;
  if (cl_max < 0) {
    cl_max = 0;
    if (cudaFuncSetAttribute(small_persistent_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
        cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(GB);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxPotentialClusterSize(&n, small_persistent_kernel<true>, &q) == cudaSuccess) cl_max = n;
    }
    cudaGetLastError();
  }
  if (cl_env && cl_max >= 2 && total_vb <= 8 * cl_max) {
    cudaLaunchConfig_t cfg = {};
    const int n = std::min(cl_max, total_vb);
    cfg.gridDim = dim3(n);
    cfg.blockDim = dim3(GB);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = n;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, small_persistent_kernel<true>, A);
  }
  const int grid = std::max(1, std::min(small_persistent_grid(), total_vb));
  void* args[] = {const_cast<SmallArgs*>(&A)};
  return cudaLaunchCooperativeKernel((void*)small_persistent_kernel<false>, dim3(grid), dim3(GB), args, 0, s);
}

// ---- cluster-resident controller for small all-FOM groups (c1) ---------------------------------------------
// The persistent controller above keeps the state in global memory, so each of its phases is a chain of L2 round
// trips.  Here the whole group lives on chip, in one thread-block cluster: every CTA holds a replica of every
// subdomain's stencil input X (the checkpoint q with the current Schwarz values) and of the checkpoint u (the
// previous step's X) in its shared memory, computes every transfer itself into its own replica (a few hundred
// nodes: cheaper than exchanging them), and advances a contiguous range of nodes of every subdomain (its own W,
// W' and Q' in shared memory).  The cluster exchanges only (a) the CTAs' norm partials once per sweep (DSMEM, one
// cluster barrier) and (b) once per controller step the new checkpoint q of every CTA's nodes into every replica
// (DSMEM stores, one cluster barrier).  The two X replicas alternate by step parity, the three W buffers by role.
// Per node the arithmetic is gather_body's (class-table stencil, the same FMA order, the same finish) and per
// destination DOF small_xfer's, so the states are bitwise those of the graph path; only the summation order of
// the convergence norm differs (every CTA sums the partials in rank order, so all take the same decision).
constexpr int RB = 512;  // threads per CTA (4 lanes per node: 128 nodes per pass)

__device__ __forceinline__ int res_chunk(int n, int nc) { return (n + nc - 1) / nc; }

template <int NTH>
__device__ __forceinline__ double2 cta_sum2(double num, double den, double* red) {
  num = warp_sum(num);
  den = warp_sum(den);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[2 * w] = num;
    red[2 * w + 1] = den;
  }
  __syncthreads();
  double a = 0.0, b = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < NTH / 32; ++q) {
      a += red[2 * q];
      b += red[2 * q + 1];
    }
  return make_double2(a, b);
}

__device__ __forceinline__ void res_step_begin(const Ctl& C, int step) {
  C.active[0] = 1;
  C.iters[0] = 0;
  C.flags[0] = 1;
  C.flags[1] = 0;
  *C.n_dev = 0;
  *C.step_dev = step;
}

// in-range test of a neighbour offset o in {-1, 0, 1} for a node of axis class c (0 low face, 2 high face)
__device__ __forceinline__ bool res_in(int c, int o) { return !((c == 0 && o < 0) || (c == 2 && o > 0)); }

constexpr int RGRP = RB / 96;  // node groups of 3 warps per pass (5: 160 nodes; the 16th warp idles)
__global__ void __launch_bounds__(RB, 1) small_resident_kernel(const __grid_constant__ SmallArgs A) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ double sfr[RGRP][3][3][32];  // the planes' forces of a pass (11.5 KB static)
  cg::cluster_group cl = cg::this_cluster();
  const int NC = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const Ctl& C = A.ctl;
  // shared memory: X replicas [2][xtot] | per subdomain W[3 buffers][3][chunk], Q'[3][chunk] | per owned slot
  // (offset, class | free mask << 5 | mass index << 8) | partials [2] | block scratch | flag | class tables |
  // transfer maps (idx [8n], out [3n], xi [3n])
  int xoff[SMALL_MAX_SD], woff[SMALL_MAX_SD], chunk[SMALL_MAX_SD], cum[SMALL_MAX_SD + 1];
  int xtot = 0, wtot = 0;
  cum[0] = 0;
  for (int i = 0; i < A.n_sd; ++i) {
    const Geom& g = A.s[i].L.g;
    xoff[i] = xtot;
    xtot += (int)g.total;
    chunk[i] = res_chunk(g.nn[0] * g.nn[1] * g.nn[2], NC);
    woff[i] = wtot;
    wtot += 12 * chunk[i];
    cum[i + 1] = cum[i] + chunk[i];
  }
  const int nslot = cum[A.n_sd];
  double* Xb[2] = {rsm, rsm + xtot};
  double* Wb = rsm + 2 * xtot;
  int2* meta = reinterpret_cast<int2*>(Wb + wtot);
  double2* cpart = reinterpret_cast<double2*>(meta + (nslot + 1) / 2 * 2);  // [2] (16-byte aligned)
  double* red = reinterpret_cast<double*>(cpart + 2);          // [2 * RB / 32]
  int* flag = reinterpret_cast<int*>(red + 2 * (RB / 32));     // [4]
  double* csm = reinterpret_cast<double*>(flag + 4);
  const double* coefp[SMALL_MAX_SD];
  for (int i = 0; i < A.n_sd; ++i) {
    coefp[i] = A.s[i].L.coef;
    if (A.res_coef_smem) {
      double* dst = csm + (size_t)i * NCLASS * 27 * 9;
      for (int t = tid; t < NCLASS * 27 * 9; t += RB) dst[t] = A.s[i].L.coef[t];
      coefp[i] = dst;
    }
  }
  // the transfer maps (read every sweep) in shared memory
  unsigned char* mp = reinterpret_cast<unsigned char*>(csm + (A.res_coef_smem ? (size_t)A.n_sd * NCLASS * 27 * 9 : 0));
  SmallMap maps[SMALL_MAX_SD][6];
  for (int i = 0; i < A.n_sd; ++i)
    for (int mi = 0; mi < A.s[i].n_maps; ++mi) {
      const SmallMap& m = A.s[i].maps[mi];
      double* xi = reinterpret_cast<double*>(mp);
      int* idx = reinterpret_cast<int*>(xi + 3 * m.n);
      int* out = idx + 8 * m.n;
      for (int t = tid; t < 3 * m.n; t += RB) {
        xi[t] = m.xi[t];
        out[t] = m.out[t];
      }
      for (int t = tid; t < 8 * m.n; t += RB) idx[t] = m.idx[t];
      maps[i][mi] = SmallMap{m.n, m.src, idx, out, xi};
      mp += ((size_t)3 * m.n * 8 + (size_t)11 * m.n * 4 + 15) / 16 * 16;
    }

  // load the replicas (X = q of the checkpoint, U = u of the checkpoint), this CTA's W and its slots' metadata
  for (int i = 0; i < A.n_sd; ++i) {
    const SmallSub& d = A.s[i];
    const Geom& g = d.L.g;
    const double* q0 = d.st[d.cur0][0];
    const double* u0 = d.st[1 - d.cur0][0];
    for (long long t = tid; t < g.total; t += RB) {
      Xb[0][xoff[i] + t] = q0[t];
      Xb[1][xoff[i] + t] = u0[t];
    }
    const int n = g.nn[0] * g.nn[1] * g.nn[2];
    for (int l = tid; l < chunk[i]; l += RB) {
      const int t = rank * chunk[i] + l;
      int2 mt = make_int2(-1, 0);
      if (t < n) {
        const int ii = t % g.nn[0], jj = (t / g.nn[0]) % g.nn[1], kk = t / (g.nn[0] * g.nn[1]);
        const int cx = axis_class(ii, g.nn[0]), cy = axis_class(jj, g.nn[1]), cz = axis_class(kk, g.nn[2]);
        const int im = (cx == 1 ? 1 : 0) + (cy == 1 ? 2 : 0) + (cz == 1 ? 4 : 0);
        mt = make_int2((int)gidx(g, ii, jj, kk), (cx + 3 * (cy + 3 * cz)) | ((int)free_mask(g, d.L.f, ii, jj, kk) << 5) |
                                                     (im << 8));
#pragma unroll
        for (int c = 0; c < 3; ++c) Wb[woff[i] + c * chunk[i] + l] = d.st[d.cur0][1][c * g.npad + mt.x];
      }
      meta[cum[i] + l] = mt;
    }
  }
  // controller state lives in rank 0's registers; the global copies are only written
  int step = 0, active = 1;
  if (rank == 0 && tid == 0) {
    step = *C.step_dev + 1;
    res_step_begin(C, step);
  }
  int ck = 0;    // W buffer of the checkpoint (buffers 0..2, each [3][chunk])
  int kpar = 0;  // X replica of the current step (the other one holds u of the checkpoint)
  cl.sync();
#ifdef OSAM_RES_PROF
  long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t_0 = clock64();
#define RES_T(q) if (tid == 0 && rank == 0) { const long long t_ = clock64(); tp[q] += t_ - t_0; t_0 = t_; }
#else
#define RES_T(q)
#endif
  for (int k = 0; k < A.n_steps; ++k) {
    double* Xc = Xb[kpar];
    const double* Xu = Xb[1 - kpar];
    int wo = ck;
    for (int n = 1; n <= A.max_iters; ++n) {
      const bool first = n == 1;
      const int wp = wo;            // W' of iterate n - 1 (unused at n = 1)
      wo = (ck + 1 + (n & 1)) % 3;  // W' of iterate n: alternates between the two non-checkpoint buffers
      // K2 in sweep order into this CTA's replica (a later destination reads iterate n of an earlier source)
      for (int i = 0; i < A.n_sd; ++i) {
        const int nm = A.s[i].n_maps;
        for (int mi = 0; mi < nm; ++mi) {
          const SmallMap& m = maps[i][mi];
          const bool newest = (m.src < i) || !first;
          const double* field = (newest ? Xc : Xu) + xoff[m.src];
          const int cs = (int)A.s[m.src].L.g.npad;
          for (int t = tid; t < 3 * m.n; t += RB) {
            const int p = t / 3, cc = t - 3 * p;
            const int o = m.out[t];
            if (o < 0) continue;
            const double xx = m.xi[3 * p], yy = m.xi[3 * p + 1], zz = m.xi[3 * p + 2];
            const double* sb = field + cc * cs;
            const int* ix = m.idx + 8 * p;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const double w = ((q & 1) ? xx : 1.0 - xx) * ((q & 2) ? yy : 1.0 - yy) * ((q & 4) ? zz : 1.0 - zz);
              acc = fma(w, sb[ix[q]], acc);
            }
            Xc[xoff[i] + o] = acc;
          }
        }
        if (nm) __syncthreads();
      }
      RES_T(0);
      // K1S on this CTA's nodes of every subdomain, gather_body's arithmetic and layout: groups of 32 nodes, warp
      // 3 g + o gathers the plane oz = o - 1 of group g (one class-table offset per warp), the planes meet in
      // shared memory and the group's first warp sums them in the order (-1 + 0) + 1 and finishes
      double num = 0.0, den = 0.0;
      const int lane = tid & 31, grp = (tid >> 5) / 3, o = (tid >> 5) % 3;
      for (int u0 = 0; u0 < nslot; u0 += RGRP * 32) {
        const int u = u0 + grp * 32 + lane;
        int i = 0;
        while (i + 1 < A.n_sd && u >= cum[i + 1]) ++i;
        const int2 mt = (grp < RGRP && u < nslot) ? meta[u] : make_int2(-1, 0);
        const bool valid = mt.x >= 0;
        const int cls = mt.y & 31, cx = cls % 3, cy = (cls / 3) % 3, cz = cls / 9;
        const SmallSub& d = A.s[i];
        const Geom& g = d.L.g;
        const double* X = Xc + xoff[i];
        const int np = (int)g.npad, px = g.px, pl = (int)g.plane;
        double f[3] = {0.0, 0.0, 0.0};
        const int oz = o - 1;
        if (valid && res_in(cz, oz)) {
          const double* coef = coefp[i] + (size_t)cls * 27 * 9;
#pragma unroll
          for (int oy = -1; oy <= 1; ++oy) {
            if (!res_in(cy, oy)) continue;
#pragma unroll
            for (int ox = -1; ox <= 1; ++ox) {
              if (!res_in(cx, ox)) continue;
              const int q = mt.x + ox + px * oy + pl * oz;
              const double x[3] = {X[q], X[np + q], X[2 * np + q]};
              const double* cb = coef + ((ox + 1) + 3 * ((oy + 1) + 3 * (oz + 1))) * 9;
#pragma unroll
              for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int dd = 0; dd < 3; ++dd) f[c] = fma(cb[c * 3 + dd], x[dd], f[c]);
            }
          }
        }
        if (grp < RGRP)
#pragma unroll
          for (int c = 0; c < 3; ++c) sfr[grp][o][c][lane] = f[c];
        __syncthreads();
        if (grp < RGRP && o == 0)
#pragma unroll
          for (int c = 0; c < 3; ++c) f[c] = (sfr[grp][0][c][lane] + sfr[grp][1][c][lane]) + sfr[grp][2][c][lane];
        const int sub = o;
        if (valid && sub == 0) {
          const unsigned fm = (unsigned)(mt.y >> 5) & 7u;
          const FomLaunch& L = d.L;
          const double inv_m = L.inv_mass[(mt.y >> 8) & 7];
          double* W = Wb + woff[i];
          const int ch = chunk[i], l = u - cum[i];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double x = X[c * np + mt.x];
            double wn = 0.0, qn = x;
            if ((fm >> c) & 1) {
              const double w0 = W[(ck * 3 + c) * ch + l];
              const double an = -f[c] * inv_m;
              wn = fma(L.cw, an, w0);
              qn = fma(L.cq, wn, x);
              const double w = fma(L.dt, fma(L.cv, an, w0), x);
              if (!first) {
                const double dl = 0.5 * L.dt * (wn - W[(wp * 3 + c) * ch + l]);
                num = fma(dl, dl, num);
                den = fma(w, w, den);
              }
            }
            W[(wo * 3 + c) * ch + l] = wn;
            W[(9 + c) * ch + l] = qn;
          }
        }
        __syncthreads();  // sfr is reused by the next pass
      }
      RES_T(1);
      // the CTA's (num, den), then the cluster's, summed by the same butterfly in every CTA (the same decision
      // everywhere)
      const double2 mine = cta_sum2<RB>(num, den, red);
      if (tid == 0) cpart[n & 1] = mine;
      RES_T(2);
      cl.sync();
      RES_T(3);
      if (tid < 32) {
        double2 v = make_double2(0.0, 0.0);
        if (tid < NC) v = *cl.map_shared_rank(cpart + (n & 1), tid);
        double sn = v.x, sd = v.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sn += __shfl_xor_sync(0xffffffffu, sn, o);
          sd += __shfl_xor_sync(0xffffffffu, sd, o);
        }
        bool conv = false, bad = false;
        if (n >= A.min_iters) {
          bad = !isfinite(sn) || !isfinite(sd);
          conv = (sn == 0.0) || (sn < A.tol_rel * A.tol_rel * sd);
          if (A.tol_abs > 0.0) conv = conv || (sn < A.tol_abs * A.tol_abs);
        }
        const int go = !conv && !bad && n < A.max_iters;
        if (rank == 0 && tid == 0) {  // controller state (as small_persistent_kernel's K3), stores only
          C.iters[0] = n;
          if (n >= A.min_iters) {
            C.numden[0] = sn;
            C.numden[1] = sd;
            if (C.trace && n <= C.trace_T) {  // convergence trace (osam_set_conv_trace), B = 1
              double* tr = C.trace + 2 * ((long long)(step - 1) * C.trace_T + (n - 1));
              tr[0] = sn;
              tr[1] = sd;
            }
            if (bad) {
              C.flags[1] = 1;
              C.sticky[0] = 1;
            }
          }
          if (conv) active = 0;
          C.active[0] = active;
          *C.n_dev = n;
          C.flags[0] = active;
          if (C.iters_all) C.iters_all[step - 1] = n;
          if (active && n >= A.max_iters) C.sticky[1] = 1;
          if (!go && k + 1 < A.n_steps) {
            ++step;
            active = 1;
            res_step_begin(C, step);
          }
        }
        if (tid == 0) flag[0] = go;
      }
      __syncthreads();
      RES_T(4);
      if (!flag[0]) break;
    }
    // commit: the new checkpoint q (Q' of the last iterate) of this CTA's nodes into every replica's other buffer
    // (which held u of the old checkpoint, no longer read); the last iterate's W' becomes the checkpoint w
    double* Xn = Xb[1 - kpar];
    for (int i = 0; i < A.n_sd; ++i) {
      const int ch = chunk[i], np = (int)A.s[i].L.g.npad;
      const double* QN = Wb + woff[i] + 9 * ch;
      for (int e = tid; e < 3 * ch; e += RB) {
        const int c = e / ch, l = e - c * ch;
        const int ofs = meta[cum[i] + l].x;
        if (ofs < 0) continue;
        const double v = QN[e];
        double* dst = Xn + xoff[i] + c * np + ofs;
        for (int r = 0; r < NC; ++r) *cl.map_shared_rank(dst, r) = v;
      }
    }
    ck = wo;
    kpar ^= 1;
    RES_T(5);
    cl.sync();
    RES_T(6);
  }
#ifdef OSAM_RES_PROF
  if (tid == 0 && rank == 0)
    printf("RESPROF NC %d steps %d cycles: xfer %lld stencil %lld ctasum %lld clsync %lld decide %lld commit %lld commitsync %lld\n",
           NC, A.n_steps, tp[0], tp[1], tp[2], tp[3], tp[4], tp[5], tp[6]);
#endif
  // write back: the checkpoint buffer gets q (this CTA's nodes) and w, the spare buffer's q slot u (R30)
  for (int i = 0; i < A.n_sd; ++i) {
    const SmallSub& d = A.s[i];
    const int cbf = (A.n_steps & 1) ? 1 - d.cur0 : d.cur0;
    const Geom& g = d.L.g;
    const int ch = chunk[i];
    for (int e = tid; e < 3 * ch; e += RB) {
      const int c = e / ch, l = e - c * ch;
      const int ofs = meta[cum[i] + l].x;
      if (ofs < 0) continue;
      const long long o = c * g.npad + ofs;
      d.st[cbf][0][o] = Xb[kpar][xoff[i] + o];
      d.st[1 - cbf][0][o] = Xb[1 - kpar][xoff[i] + o];
      d.st[cbf][1][o] = Wb[woff[i] + (ck * 3 + c) * ch + l];
    }
  }
}

// Launch of the cluster-resident controller; cudaErrorNotSupported when the group does not fit one cluster's
// shared memory (or clusters of >= 2 CTAs are unavailable): the caller then uses small_persistent_kernel.
cudaError_t launch_small_resident(const SmallArgs& A, cudaStream_t s) {
  if (getenv("OSAM_SMALL_RESIDENT") && getenv("OSAM_SMALL_RESIDENT")[0] == '0') return cudaErrorNotSupported;
  static int cl_max = -1;
  constexpr int SMEM_MAX = 227 * 1024 - (int)sizeof(double) * RGRP * 9 * 32;  // dynamic; the pass buffer is static
  if (cl_max < 0) {
    cl_max = 0;
    if (cudaFuncSetAttribute(small_resident_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess &&
        cudaFuncSetAttribute(small_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX) ==
            cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(RB);
      q.dynamicSmemBytes = SMEM_MAX;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxPotentialClusterSize(&n, small_resident_kernel, &q) == cudaSuccess) cl_max = n;
    }
    cudaGetLastError();
  }
  if (cl_max < 2) return cudaErrorNotSupported;
  int NC = std::min(cl_max, 16);
  if (const char* e = getenv("OSAM_RESIDENT_NC")) NC = std::max(2, std::min(NC, atoi(e)));  // A/B of the cluster size
  long long xtot = 0, wtot = 0;
  for (int i = 0; i < A.n_sd; ++i) {
    const Geom& g = A.s[i].L.g;
    xtot += g.total;
    wtot += 12LL * (((long long)g.nn[0] * g.nn[1] * g.nn[2] + NC - 1) / NC);
  }
  long long nslot = 0, msize = 0;
  for (int i = 0; i < A.n_sd; ++i) {
    const Geom& g = A.s[i].L.g;
    nslot += ((long long)g.nn[0] * g.nn[1] * g.nn[2] + NC - 1) / NC;
    for (int mi = 0; mi < A.s[i].n_maps; ++mi) msize += (24LL * A.s[i].maps[mi].n + 44LL * A.s[i].maps[mi].n + 15) / 16 * 16;
  }
  long long smem = 8 * (2 * xtot + wtot) + 8 * ((nslot + 1) / 2 * 2) + 16LL * 2 + 8LL * 2 * (RB / 32) + 16 + msize;
  if (smem > SMEM_MAX) return cudaErrorNotSupported;
  SmallArgs B = A;
  const long long csize = 8LL * NCLASS * 27 * 9 * A.n_sd;
  B.res_coef_smem = smem + csize <= SMEM_MAX && !(getenv("OSAM_RESIDENT_COEF") && getenv("OSAM_RESIDENT_COEF")[0] == '0');
  if (B.res_coef_smem) smem += csize;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NC);
  cfg.blockDim = dim3(RB);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = NC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, small_resident_kernel, B);
}

void launch_fom_advance_nl(const FomLaunch& L, cudaStream_t s, int* launches) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fom_nl_kernel<OSAM_SVK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nl::SMEM);
    cudaFuncSetAttribute(fom_nl_kernel<OSAM_NEOHOOKEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nl::SMEM);
    attr = true;
  }
  const dim3 block(nl::NTN);
  if (L.material == OSAM_SVK)
    fom_nl_kernel<OSAM_SVK><<<nl_ctas(L.g), block, nl::SMEM, s>>>(L);
  else
    fom_nl_kernel<OSAM_NEOHOOKEAN><<<nl_ctas(L.g), block, nl::SMEM, s>>>(L);
  debug_check("fom_nl_kernel", s);
  ++*launches;
}

void launch_fom_xlast(const FomLaunch& L, cudaStream_t s, int* launches) {
  if (L.material != OSAM_LINEAR || small_fom(L.g)) return;
  const int sh = k1_shape(L.g, L.f);
  if (!(sh == 1 ? k1b::xlast_excluded(L.g, L.f) : sh == 2 ? k1c::xlast_excluded(L.g, L.f) : k1a::xlast_excluded(L.g, L.f)))
    return;
  xlast_copy_kernel<<<cdiv((long long)L.g.nn[1] * L.g.nn[2], 128 * XL_PER), 128, 0, s>>>(L);
  debug_check("xlast_copy_kernel", s);
  ++*launches;
}

void launch_fom_advance(const FomLaunch& L, const InteriorStencil& st, const CUtensorMap* tmx,
                        const CUtensorMap* tmw, const CUtensorMap* tmwp, cudaStream_t s, int* launches,
                        bool with_xlast) {
  if (L.material != OSAM_LINEAR) {  // SVK / Neohookean: NL1 (no stencil, no TMA maps)
    launch_fom_advance_nl(L, s, launches);
    return;
  }
  if (small_fom(L.g)) {  // K1S: one gather pass over every node
    launch_k(fom_gather_kernel, dim3(cdiv((long long)L.g.nn[0] * L.g.nn[1] * L.g.nn[2], GNODES)), dim3(GB), 0, s, L);
    debug_check("fom_gather_kernel", s);
    ++*launches;
    return;
  }
  switch (k1_shape(L.g, L.f)) {
    case 1: k1b::launch_tiled(L, st, tmx, tmw, tmwp, s); break;
    case 2: k1c::launch_tiled(L, st, tmx, tmw, tmwp, s); break;
    default: k1a::launch_tiled(L, st, tmx, tmw, tmwp, s);
  }
  ++*launches;
  if (with_xlast) launch_fom_xlast(L, s, launches);
}

int make_field_tmap(const Geom& g, const Faces& f, double* array, bool halo, CUtensorMap* out) {
  switch (k1_shape(g, f)) {
    case 1: return k1b::make_tmap(g, array, halo, out);
    case 2: return k1c::make_tmap(g, array, halo, out);
    default: return k1a::make_tmap(g, array, halo, out);
  }
}

void launch_fom_pack(const Geom& g, const double* src, double* dst, long long n, cudaStream_t s) {
  pack_kernel<<<cdiv(n, 256), 256, 0, s>>>(g, src, dst, n);
  debug_check("pack_kernel", s);
}

void launch_fom_unpack(const Geom& g, const double* src, double* dst, long long n, cudaStream_t s) {
  unpack_kernel<<<cdiv(n, 256), 256, 0, s>>>(g, src, dst, n);
  debug_check("unpack_kernel", s);
}

void launch_fom_zero_constrained(const Geom& g, const Faces& f, double* u, double* w, cudaStream_t s) {
  zero_constrained_kernel<<<cdiv(surface_count(g), 256), 256, 0, s>>>(g, f, u, w);
  debug_check("zero_constrained_kernel", s);
}

}  // namespace osam

