// K1: fused FOM advance -- explicit Newmark (beta = 0, gamma = 1/2) step of a hex8
// linear-elastic box subdomain with lumped mass (A.1 P:L1934-1947):
//
//   u* = u + dt v + dt^2/2 a  on free DOFs, 0 on Dirichlet DOFs, s on Schwarz DOFs
//   f  = K u*                 (matrix-free 27-point merged hex8 stencil, 153 nonzeros/node)
//   a' = -f / m_L ,  v' = v + dt/2 (a + a')   on free DOFs (v' = a' = 0 on constrained DOFs)
//   partial sums of ||(u*-u_prev) + dt (v'-v_prev)||^2 and ||u* + dt v'||^2 (eq:conv_criterion)
//
// Two kernels make one K1:
//   * the tiled kernel covers every node with 1 <= i <= nx-1 (all j, k).  A block owns a
//     TX x TY tile in (x, y) and a chunk of ZC node planes; it streams the checkpoint planes
//     (u, v, a; tile + one-node halo) with 4D TMA loads into a 3-deep mbarrier ring, forms
//     the predictor once per staged position, and accumulates each staged plane into the
//     forces of node planes m-1, m, m+1 held in registers.  A warp is one x-row, so the
//     boundary class in (y, z) is warp-uniform: interior rows use the 153-coefficient stencil
//     held in the kernel-parameter constant bank, face rows read their class table.
//   * the x-face kernel covers i = 0 and i = nx (a node per thread, class table).
// No atomics; every sum has a fixed order, so results are bitwise repeatable.
#include "osam_internal.h"

namespace osam {

namespace {

constexpr int TX = 32;
constexpr int TY = 8;
constexpr int ZC = 16;
constexpr int XF_BLOCK = 128;

__device__ __forceinline__ long long gidx(const Geom& g, int i, int j, int k) {
  return i + (long long)g.px * (j + (long long)g.nn[1] * k);
}

// DOF code of (i,j,k,c): Dirichlet > Schwarz (lowest Schwarz face holding the node) > free.
__device__ __forceinline__ int dof_code(const Geom& g, const Faces& F, int i, int j, int k, int c, double* sv) {
  const int idx[3] = {i, j, k};
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const bool on = idx[ax] == ((f & 1) ? g.nn[ax] - 1 : 0);
    if (on && ((F.dir[f] >> c) & 1)) return DOF_DIRICHLET;
  }
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const bool on = idx[ax] == ((f & 1) ? g.nn[ax] - 1 : 0);
    if (on && F.sw[f]) {
      const int o0 = ax == 0 ? 1 : 0;
      const int o1 = ax == 2 ? 1 : 2;
      const long long fi = idx[o0] + (long long)g.nn[o0] * idx[o1];
      *sv = F.s[f][c * (long long)F.nface[f] + fi];
      return DOF_SCHWARZ;
    }
  }
  return DOF_FREE;
}

__device__ __forceinline__ double predict(double u, double v, double a, double dt) {
  return fma(0.5 * dt * dt, a, fma(dt, v, u));
}

__device__ __forceinline__ double predict_bc(const Geom& g, const Faces& F, int i, int j, int k, int c, double u,
                                             double v, double a, double dt) {
  double sv = 0.0;
  const int code = dof_code(g, F, i, j, k, c, &sv);
  return code == DOF_FREE ? predict(u, v, a, dt) : (code == DOF_SCHWARZ ? sv : 0.0);
}

__device__ __forceinline__ int axis_class(int idx, int nn) { return idx == 0 ? 0 : (idx == nn - 1 ? 2 : 1); }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Fixed-order block reduction of (num, den) -> partial[slot].
template <int NT>
__device__ __forceinline__ void block_partial(double num, double den, double2* partial, int slot) {
  __shared__ double red[2][NT / 32];
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
    for (int w = 0; w < NT / 32; ++w) {
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

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int c,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(c), "r"(smem_u32(bar))
      : "memory");
}

constexpr int PX = TX + 2;
constexpr int PY = TY + 2;
constexpr int PLANE = PX * PY;                             // positions per staged plane
constexpr int NSTAGE = 3;                                  // TMA ring depth (2 planes in flight)
constexpr int ARR_BYTES = 3 * PLANE * 8;                   // one array (x,y,z comps) of one plane
constexpr int ARR_STRIDE = (ARR_BYTES + 127) / 128 * 128;  // 128-B aligned TMA destinations
constexpr int STAGE_BYTES = 3 * ARR_STRIDE;                // u, v, a
constexpr int USTAR_BYTES = 3 * PLANE * 8;
constexpr int SMEM_TILED = NSTAGE * STAGE_BYTES + 2 * USTAR_BYTES + 64;

// Interior-row stencil: off-diagonal blocks (c != d) vanish unless o_c != 0 and o_d != 0.
template <int OZ, int OX, int OY>
__device__ __forceinline__ void stencil_acc(double acc[3], const double w[3], const InteriorStencil& S) {
  constexpr int o[3] = {OX - 1, OY - 1, OZ - 1};
  constexpr int off = OX + 3 * (OY + 3 * OZ);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (c == d || (o[c] != 0 && o[d] != 0)) acc[c] = fma(S.c[off * 9 + c * 3 + d], w[d], acc[c]);
    }
  }
}

template <int OZ>
__device__ __forceinline__ void plane_acc(double acc[3], const double* us, int tx, int ty, const InteriorStencil& S) {
#define OSAM_TAP(OX, OY)                                           \
  {                                                                \
    const int q = (ty + OY) * PX + tx + OX;                        \
    const double w[3] = {us[q], us[PLANE + q], us[2 * PLANE + q]}; \
    stencil_acc<OZ, OX, OY>(acc, w, S);                            \
  }
  OSAM_TAP(0, 0) OSAM_TAP(1, 0) OSAM_TAP(2, 0)
  OSAM_TAP(0, 1) OSAM_TAP(1, 1) OSAM_TAP(2, 1)
  OSAM_TAP(0, 2) OSAM_TAP(1, 2) OSAM_TAP(2, 2)
#undef OSAM_TAP
}

// Face rows (warp-uniform class): full 3x3 blocks from the class table (L1 broadcast).
template <int OZ>
__device__ __forceinline__ void plane_acc_class(double acc[3], const double* us, int tx, int ty,
                                                const double* __restrict__ cls_coef) {
#pragma unroll
  for (int oy = 0; oy < 3; ++oy) {
#pragma unroll
    for (int ox = 0; ox < 3; ++ox) {
      const int q = (ty + oy) * PX + tx + ox;
      const double w[3] = {us[q], us[PLANE + q], us[2 * PLANE + q]};
      const double* cb = cls_coef + (ox + 3 * (oy + 3 * OZ)) * 9;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[c] = fma(__ldg(cb + c * 3 + d), w[d], acc[c]);
    }
  }
}

template <int OZ>
__device__ __forceinline__ void target_acc(double acc[3], const double* us, int tx, int ty, int cy, int cz,
                                           const InteriorStencil& S, const double* coef) {
  if (cy == 1 && cz == 1)
    plane_acc<OZ>(acc, us, tx, ty, S);
  else
    plane_acc_class<OZ>(acc, us, tx, ty, coef + (size_t)(1 + 3 * (cy + 3 * cz)) * 27 * 9);
}

__global__ void __launch_bounds__(TX* TY, 2)
    fom_tiled_kernel(const FomLaunch L, const InteriorStencil S, const __grid_constant__ CUtensorMap tu,
                     const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap ta) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* raw = reinterpret_cast<double*>(smem);
  double* ust = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + NSTAGE * STAGE_BYTES + 2 * USTAR_BYTES);
  const Geom& g = L.g;
  const int nx = g.nn[0] - 1, ny = g.nn[1] - 1, nz = g.nn[2] - 1;
  const long long np = g.npad;
  const int tx = threadIdx.x, ty = threadIdx.y, t = ty * TX + tx;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY - 1;  // node coordinates of staged position (0,0)
  const int i = x0 + 1 + tx, j = y0 + 1 + ty;
  const bool active = (i <= nx - 1) && (j <= ny);
  const int cy = axis_class(j, g.nn[1]);  // warp-uniform (a warp is one x-row)
  const int kbeg = blockIdx.z * ZC;
  const int kend = min(kbeg + ZC - 1, nz);
  const int nplanes = kend - kbeg + 3;
  const double dt = L.dt, hdt = 0.5 * dt;
  const int qo = (ty + 1) * PX + (tx + 1);

  if (t == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int it) {
    const int s = it % NSTAGE;
    const int m = kbeg - 1 + it;
    double* dst = raw + (size_t)s * (STAGE_BYTES / 8);
    mbar_expect_tx(&bar[s], 3 * ARR_BYTES);
    tma_load_4d(dst, &tu, x0, y0, m, 0, &bar[s]);
    tma_load_4d(dst + ARR_STRIDE / 8, &tv, x0, y0, m, 0, &bar[s]);
    tma_load_4d(dst + 2 * (ARR_STRIDE / 8), &ta, x0, y0, m, 0, &bar[s]);
  };
  if (t == 0) {
    issue(0);
    if (nplanes > 1) issue(1);
  }

  double accA[3] = {0.0, 0.0, 0.0}, accB[3] = {0.0, 0.0, 0.0}, accC[3] = {0.0, 0.0, 0.0};
  double pu[3] = {0.0, 0.0, 0.0}, pv[3] = {0.0, 0.0, 0.0}, pa[3] = {0.0, 0.0, 0.0};  // own node, plane m-1
  double num = 0.0, den = 0.0;

  for (int it = 0; it < nplanes; ++it) {
    const int m = kbeg - 1 + it;
    const int s = it % NSTAGE;
    const bool bplane = (m == 0) || (m == nz);
    const int kf = m - 1;  // node plane finished in this iteration
    const bool fin = active && (kf >= kbeg) && (kf <= kend);
    // previous Schwarz iterate of plane m-1 (convergence norm): issued before the wait
    double qu[3] = {0.0, 0.0, 0.0}, qv[3] = {0.0, 0.0, 0.0};
    if (fin && L.with_norm) {
      const long long id = gidx(g, i, j, kf);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        qu[c] = L.u1[c * np + id];
        qv[c] = L.v1[c * np + id];
      }
    }
    mbar_wait(&bar[s], (unsigned)((it / NSTAGE) & 1));
    const double* ru = raw + (size_t)s * (STAGE_BYTES / 8);
    const double* rv = ru + ARR_STRIDE / 8;
    const double* ra = rv + ARR_STRIDE / 8;
    double* us = ust + (it & 1) * 3 * PLANE;
    const bool mval = m >= 0 && m <= nz;
    for (int q = t; q < PLANE; q += TX * TY) {
      const int ii = x0 + q % PX, jj = y0 + q / PX;
      double w[3] = {0.0, 0.0, 0.0};
      if (mval && ii <= nx && jj >= 0 && jj <= ny) {
        const bool bnd = bplane || ii == 0 || ii == nx || jj == 0 || jj == ny;
        if (bnd) {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            w[c] = predict_bc(g, L.f, ii, jj, m, c, ru[c * PLANE + q], rv[c * PLANE + q], ra[c * PLANE + q], dt);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) w[c] = predict(ru[c * PLANE + q], rv[c * PLANE + q], ra[c * PLANE + q], dt);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) us[c * PLANE + q] = w[c];
    }
    double cv[3], ca[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cv[c] = rv[c * PLANE + qo];
      ca[c] = ra[c * PLANE + qo];
    }
    __syncthreads();
    if (t == 0 && it + 2 < nplanes) issue(it + 2);  // refills the stage of plane m-1 (consumed)
    double cu[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) cu[c] = us[c * PLANE + qo];
    if (active) {
      if (m + 1 >= kbeg && m + 1 <= kend)  // node plane m+1, oz = -1
        target_acc<0>(accA, us, tx, ty, cy, axis_class(m + 1, g.nn[2]), S, L.coef);
      if (m >= kbeg && m <= kend)  // node plane m, oz = 0
        target_acc<1>(accB, us, tx, ty, cy, axis_class(m, g.nn[2]), S, L.coef);
      if (fin) {  // node plane m-1, oz = +1
        const int cz = axis_class(kf, g.nn[2]);
        target_acc<2>(accC, us, tx, ty, cy, cz, S, L.coef);
        const long long id = gidx(g, i, j, kf);
        const bool face_row = cy != 1 || cz != 1;
        const double inv_m = 1.0 / (L.mass_e * 2.0 * (cy == 1 ? 2.0 : 1.0) * (cz == 1 ? 2.0 : 1.0));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double sv;
          const bool free_dof = !face_row || dof_code(g, L.f, i, j, kf, c, &sv) == DOF_FREE;
          double an = 0.0, vn = 0.0;
          if (free_dof) {
            an = -accC[c] * inv_m;
            vn = fma(hdt, pa[c] + an, pv[c]);
            if (L.with_norm) {
              const double d = (pu[c] - qu[c]) + dt * (vn - qv[c]);
              const double w = pu[c] + dt * vn;
              num = fma(d, d, num);
              den = fma(w, w, den);
            }
          }
          L.u1[c * np + id] = pu[c];
          L.v1[c * np + id] = vn;
          L.a1[c * np + id] = an;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      accC[c] = accB[c];
      accB[c] = accA[c];
      accA[c] = 0.0;
      pu[c] = cu[c];
      pv[c] = cv[c];
      pa[c] = ca[c];
    }
  }
  const int slot = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  block_partial<TX * TY>(num, den, L.partial, slot);
}

// Nodes on the faces x = 0 and x = nx (one per thread).  Fully constrained nodes (e.g. a
// clamped or Schwarz face) need no force: u = prescribed value, v = a = 0.
__global__ void __launch_bounds__(XF_BLOCK) fom_xface_kernel(const FomLaunch L, int slot0) {
  const Geom& g = L.g;
  const long long np = g.npad;
  const long long nf = (long long)g.nn[1] * g.nn[2];
  const long long t = blockIdx.x * (long long)XF_BLOCK + threadIdx.x;
  const double dt = L.dt, hdt = 0.5 * dt;
  const int nx = g.nn[0] - 1;
  double num = 0.0, den = 0.0;
  if (t < 2 * nf) {
    const int side = t >= nf;
    const long long r = t - side * nf;
    const int i = side ? nx : 0;
    const int j = (int)(r % g.nn[1]);
    const int k = (int)(r / g.nn[1]);
    const long long id = gidx(g, i, j, k);
    int code[3];
    double own[3];
    bool any_free = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double sv = 0.0;
      code[c] = dof_code(g, L.f, i, j, k, c, &sv);
      own[c] = code[c] == DOF_SCHWARZ ? sv : 0.0;
      any_free = any_free || code[c] == DOF_FREE;
    }
    double f[3] = {0.0, 0.0, 0.0};
    if (any_free) {
      const int cl[3] = {side ? 2 : 0, axis_class(j, g.nn[1]), axis_class(k, g.nn[2])};
      const double* coef = L.coef + (size_t)(cl[0] + 3 * (cl[1] + 3 * cl[2])) * 27 * 9;
      const int oxlo = side ? -1 : 0, oxhi = side ? 0 : 1;
      for (int oz = -1; oz <= 1; ++oz) {
        const int kk = k + oz;
        if (kk < 0 || kk >= g.nn[2]) continue;
        for (int oy = -1; oy <= 1; ++oy) {
          const int jj = j + oy;
          if (jj < 0 || jj >= g.nn[1]) continue;
          for (int ox = oxlo; ox <= oxhi; ++ox) {
            const int ii = i + ox;
            if (ii < 0 || ii > nx) continue;
            const long long q = gidx(g, ii, jj, kk);
            double us[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
              us[c] = predict_bc(g, L.f, ii, jj, kk, c, __ldg(L.u0 + c * np + q), __ldg(L.v0 + c * np + q),
                                 __ldg(L.a0 + c * np + q), dt);
            if (ox == 0 && oy == 0 && oz == 0) {
#pragma unroll
              for (int c = 0; c < 3; ++c) own[c] = us[c];
            }
            const double* cb = coef + ((ox + 1) + 3 * ((oy + 1) + 3 * (oz + 1))) * 9;
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int d = 0; d < 3; ++d) f[c] = fma(__ldg(cb + c * 3 + d), us[d], f[c]);
          }
        }
      }
    }
    const double mult = (axis_class(j, g.nn[1]) == 1 ? 2.0 : 1.0) * (axis_class(k, g.nn[2]) == 1 ? 2.0 : 1.0);
    const double inv_m = 1.0 / (L.mass_e * mult);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double an = 0.0, vn = 0.0;
      if (code[c] == DOF_FREE) {
        an = -f[c] * inv_m;
        vn = fma(hdt, __ldg(L.a0 + c * np + id) + an, __ldg(L.v0 + c * np + id));
        if (L.with_norm) {
          const double up = L.u1[c * np + id], vp = L.v1[c * np + id];
          const double d = (own[c] - up) + dt * (vn - vp);
          const double w = own[c] + dt * vn;
          num = fma(d, d, num);
          den = fma(w, w, den);
        }
      }
      L.u1[c * np + id] = own[c];
      L.v1[c * np + id] = vn;
      L.a1[c * np + id] = an;
    }
  }
  block_partial<XF_BLOCK>(num, den, L.partial, slot0 + blockIdx.x);
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
  return 2 * n0 * n1 + 2 * n0 * (n2 - 2) + 2 * (n1 - 2) * (n2 - 2);
}

__global__ void pack_kernel(Geom g, const double* __restrict__ src, double* __restrict__ dst, long long n) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const long long i = p % g.nn[0], j = (p / g.nn[0]) % g.nn[1], k = p / ((long long)g.nn[0] * g.nn[1]);
  const long long q = i + g.px * (j + (long long)g.nn[1] * k);
  for (int c = 0; c < 3; ++c) dst[c * g.npad + q] = src[c * n + p];
}

__global__ void unpack_kernel(Geom g, const double* __restrict__ src, double* __restrict__ dst, long long n) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const long long i = p % g.nn[0], j = (p / g.nn[0]) % g.nn[1], k = p / ((long long)g.nn[0] * g.nn[1]);
  const long long q = i + g.px * (j + (long long)g.nn[1] * k);
  for (int c = 0; c < 3; ++c) dst[c * n + p] = src[c * g.npad + q];
}

__global__ void face_gather_kernel(Geom g, Faces F, const double* __restrict__ u) {
  const int f = blockIdx.y;
  if (!F.sw[f]) return;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= F.nface[f]) return;
  const int ax = f >> 1;
  const int o0 = ax == 0 ? 1 : 0, o1 = ax == 2 ? 1 : 2;
  int idx[3];
  idx[ax] = (f & 1) ? g.nn[ax] - 1 : 0;
  idx[o0] = (int)(t % g.nn[o0]);
  idx[o1] = (int)(t / g.nn[o0]);
  const long long q = gidx(g, idx[0], idx[1], idx[2]);
  for (int c = 0; c < 3; ++c) F.s[f][c * (long long)F.nface[f] + t] = u[c * g.npad + q];
}

__global__ void zero_constrained_kernel(Geom g, Faces F, double* u, double* v, double* a, int zero_u) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= surface_count(g)) return;
  int i, j, k;
  surface_node(g, t, &i, &j, &k);
  const long long q = gidx(g, i, j, k);
  for (int c = 0; c < 3; ++c) {
    double sv;
    const int code = dof_code(g, F, i, j, k, c, &sv);
    if (code != DOF_FREE) {
      v[c * g.npad + q] = 0.0;
      a[c * g.npad + q] = 0.0;
      if (zero_u && code == DOF_DIRICHLET) u[c * g.npad + q] = 0.0;
    }
  }
}

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

dim3 tiled_grid(const Geom& g) {
  const long long ix = g.nn[0] - 2;
  if (ix <= 0) return dim3(0, 0, 0);
  return dim3(cdiv(ix, TX), cdiv(g.nn[1], TY), cdiv(g.nn[2], ZC));
}

unsigned xface_blocks(const Geom& g) { return cdiv(2LL * g.nn[1] * g.nn[2], XF_BLOCK); }

}  // namespace

int fom_partial_slots(const Geom& g) {
  const dim3 gi = tiled_grid(g);
  return (int)((long long)gi.x * gi.y * gi.z + xface_blocks(g));
}

void launch_fom_advance(const FomLaunch& L, const InteriorStencil& st, const CUtensorMap* tm, cudaStream_t s,
                        int* launches) {
  const dim3 gi = tiled_grid(L.g);
  const int n_int = gi.x * gi.y * gi.z;
  if (n_int > 0) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(fom_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TILED);
      attr_set = true;
    }
    fom_tiled_kernel<<<gi, dim3(TX, TY), SMEM_TILED, s>>>(L, st, tm[0], tm[1], tm[2]);
    ++*launches;
  }
  fom_xface_kernel<<<xface_blocks(L.g), XF_BLOCK, 0, s>>>(L, n_int);
  ++*launches;
}

int make_state_tmaps(const Geom& g, double* const arrays[3], CUtensorMap out[3]) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return -1;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)g.px, (cuuint64_t)g.nn[1], (cuuint64_t)g.nn[2], 3};
  const cuuint64_t strides[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.plane * 8, (cuuint64_t)g.npad * 8};
  const cuuint32_t box[4] = {PX, PY, 1, 3};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int q = 0; q < 3; ++q) {
    CUresult r = encode(&out[q], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, arrays[q], dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return (int)r;
  }
  return 0;
}

void launch_fom_face_gather(const Geom& g, const Faces& f, const double* u, cudaStream_t s) {
  int nmax = 1;
  for (int q = 0; q < 6; ++q) nmax = f.nface[q] > nmax ? f.nface[q] : nmax;
  face_gather_kernel<<<dim3(cdiv(nmax, 256), 6), 256, 0, s>>>(g, f, u);
}

void launch_fom_pack(const Geom& g, const double* src, double* dst, long long n, cudaStream_t s) {
  pack_kernel<<<cdiv(n, 256), 256, 0, s>>>(g, src, dst, n);
}

void launch_fom_unpack(const Geom& g, const double* src, double* dst, long long n, cudaStream_t s) {
  unpack_kernel<<<cdiv(n, 256), 256, 0, s>>>(g, src, dst, n);
}

void launch_fom_zero_constrained(const Geom& g, const Faces& f, double* u, double* v, double* a, int zero_u,
                                 cudaStream_t s) {
  zero_constrained_kernel<<<cdiv(surface_count(g), 256), 256, 0, s>>>(g, f, u, v, a, zero_u);
}

}  // namespace osam
