// K1: fused FOM advance -- explicit Newmark (beta = 0, gamma = 1/2) step of a hex8
// linear-elastic box subdomain with lumped mass (A.1 P:L1934-1947):
//
//   u* = u + dt v + dt^2/2 a  on free DOFs, 0 on Dirichlet DOFs, s on Schwarz DOFs
//   f  = K u*                 (matrix-free 27-point merged hex8 stencil, 153 nonzeros/node)
//   a' = -f / m_L ,  v' = v + dt/2 (a + a')   on free DOFs (v' = a' = 0 on constrained DOFs)
//   partial sums of ||(u*-u_prev) + dt (v'-v_prev)||^2 and ||u* + dt v'||^2 (eq:conv_criterion)
//
// Two launches make one K1: an interior kernel (all 8 incident elements present, all DOFs
// free, one uniform stencil held in the kernel-parameter constant bank) that marches 2D
// (x,y) tiles along z with the predictor of each node plane staged in shared memory, and a
// surface kernel for the nodes on the box faces (27 boundary classes, coefficients from a
// small table).  No atomics; every sum has a fixed order, so results are bitwise repeatable.
#include "osam_internal.h"

namespace osam {

namespace {

constexpr int TX = 32;
constexpr int TY = 8;
constexpr int ZC = 16;
constexpr int SURF_BLOCK = 128;

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

// Accumulate one in-plane neighbour (ox, oy) of source plane offset OZ into acc.
// Off-diagonal blocks (c != d) of the interior stencil vanish unless o_c != 0 and o_d != 0.
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
__device__ __forceinline__ void plane_acc(double acc[3], const double (*sm)[TY + 2][TX + 2], int tx, int ty,
                                          const InteriorStencil& S) {
#define OSAM_TAP(OX, OY)                                                                     \
  {                                                                                          \
    const double w[3] = {sm[0][ty + OY][tx + OX], sm[1][ty + OY][tx + OX], sm[2][ty + OY][tx + OX]}; \
    stencil_acc<OZ, OX, OY>(acc, w, S);                                                      \
  }
  OSAM_TAP(0, 0) OSAM_TAP(1, 0) OSAM_TAP(2, 0)
  OSAM_TAP(0, 1) OSAM_TAP(1, 1) OSAM_TAP(2, 1)
  OSAM_TAP(0, 2) OSAM_TAP(1, 2) OSAM_TAP(2, 2)
#undef OSAM_TAP
}

__global__ void __launch_bounds__(TX* TY, 2) fom_interior_kernel(const FomLaunch L, const InteriorStencil S) {
  __shared__ double sm[2][3][TY + 2][TX + 2];
  const Geom& g = L.g;
  const int nx = g.nn[0] - 1, ny = g.nn[1] - 1, nz = g.nn[2] - 1;
  const long long np = g.npad;
  const int tx = threadIdx.x, ty = threadIdx.y, t = ty * TX + tx;
  const int i = 1 + blockIdx.x * TX + tx;
  const int j = 1 + blockIdx.y * TY + ty;
  const bool active = (i <= nx - 1) && (j <= ny - 1);
  const bool own_valid = (i <= nx) && (j <= ny);
  const int kbeg = 1 + blockIdx.z * ZC;
  const int kend = min(kbeg + ZC - 1, nz - 1);
  const double dt = L.dt, hdt = 0.5 * dt;
  const double inv_m = 1.0 / (8.0 * L.mass_e);

  // halo ring of the (TX+2) x (TY+2) tile: rows 0 and TY+1, columns 0 and TX+1
  int hx = -1, hy = -1;
  if (t < TX + 2) {
    hx = t;
    hy = 0;
  } else if (t < 2 * (TX + 2)) {
    hx = t - (TX + 2);
    hy = TY + 1;
  } else if (t < 2 * (TX + 2) + TY) {
    hx = 0;
    hy = 1 + t - 2 * (TX + 2);
  } else if (t < 2 * (TX + 2) + 2 * TY) {
    hx = TX + 1;
    hy = 1 + t - 2 * (TX + 2) - TY;
  }
  const int hi = blockIdx.x * TX + hx;  // node index of halo position (position 0 <-> node i0 - 1)
  const int hj = blockIdx.y * TY + hy;
  const bool hvalid = hx >= 0 && hi <= nx && hj <= ny;

  double accA[3] = {0.0, 0.0, 0.0}, accB[3] = {0.0, 0.0, 0.0}, accC[3] = {0.0, 0.0, 0.0};
  double pu[3] = {0.0, 0.0, 0.0}, pv[3] = {0.0, 0.0, 0.0}, pa[3] = {0.0, 0.0, 0.0};  // own, plane m-1
  double num = 0.0, den = 0.0;

  for (int m = kbeg - 1; m <= kend + 1; ++m) {
    const int buf = (m - kbeg + 1) & 1;
    const bool bplane = (m == 0) || (m == nz);
    double cu[3] = {0.0, 0.0, 0.0}, cv[3] = {0.0, 0.0, 0.0}, ca[3] = {0.0, 0.0, 0.0};
    if (own_valid) {
      const long long id = gidx(g, i, j, m);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cu[c] = __ldg(L.u0 + c * np + id);
        cv[c] = __ldg(L.v0 + c * np + id);
        ca[c] = __ldg(L.a0 + c * np + id);
      }
      const bool bnd = bplane || i == nx || j == ny;
      double us[3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        us[c] = bnd ? predict_bc(g, L.f, i, j, m, c, cu[c], cv[c], ca[c], dt) : predict(cu[c], cv[c], ca[c], dt);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        sm[buf][c][ty + 1][tx + 1] = us[c];
        cu[c] = us[c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) sm[buf][c][ty + 1][tx + 1] = 0.0;
    }
    if (hx >= 0) {
      double us[3] = {0.0, 0.0, 0.0};
      if (hvalid) {
        const long long id = gidx(g, hi, hj, m);
        const bool bnd = bplane || hi == 0 || hi == nx || hj == 0 || hj == ny;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double u = __ldg(L.u0 + c * np + id), v = __ldg(L.v0 + c * np + id), a = __ldg(L.a0 + c * np + id);
          us[c] = bnd ? predict_bc(g, L.f, hi, hj, m, c, u, v, a, dt) : predict(u, v, a, dt);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) sm[buf][c][hy][hx] = us[c];
    }
    __syncthreads();

    if (active) {
      const double(*p)[TY + 2][TX + 2] = sm[buf];
      if (m + 1 >= kbeg && m + 1 <= kend) plane_acc<0>(accA, p, tx, ty, S);  // node plane m+1, oz = -1
      if (m >= kbeg && m <= kend) plane_acc<1>(accB, p, tx, ty, S);          // node plane m,   oz =  0
      if (m - 1 >= kbeg && m - 1 <= kend) {                                  // node plane m-1, oz = +1
        plane_acc<2>(accC, p, tx, ty, S);
        const long long id = gidx(g, i, j, m - 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double an = -accC[c] * inv_m;
          const double vn = fma(hdt, pa[c] + an, pv[c]);
          if (L.with_norm) {
            const double up = L.u1[c * np + id], vp = L.v1[c * np + id];
            const double d = (pu[c] - up) + dt * (vn - vp);
            const double w = pu[c] + dt * vn;
            num = fma(d, d, num);
            den = fma(w, w, den);
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

__global__ void __launch_bounds__(SURF_BLOCK) fom_surface_kernel(const FomLaunch L, int slot0) {
  const Geom& g = L.g;
  const long long np = g.npad;
  const long long t = blockIdx.x * (long long)SURF_BLOCK + threadIdx.x;
  const double dt = L.dt, hdt = 0.5 * dt;
  double num = 0.0, den = 0.0;
  if (t < surface_count(g)) {
    int i, j, k;
    surface_node(g, t, &i, &j, &k);
    const int idx[3] = {i, j, k};
    int cl[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) cl[a] = idx[a] == 0 ? 0 : (idx[a] == g.nn[a] - 1 ? 2 : 1);
    const int cls = cl[0] + 3 * (cl[1] + 3 * cl[2]);
    const double* coef = L.coef + (long long)cls * 27 * 9;
    double f[3] = {0.0, 0.0, 0.0};
    double own_us[3] = {0.0, 0.0, 0.0};
    for (int oz = -1; oz <= 1; ++oz) {
      const int kk = k + oz;
      if (kk < 0 || kk >= g.nn[2]) continue;
      for (int oy = -1; oy <= 1; ++oy) {
        const int jj = j + oy;
        if (jj < 0 || jj >= g.nn[1]) continue;
        for (int ox = -1; ox <= 1; ++ox) {
          const int ii = i + ox;
          if (ii < 0 || ii >= g.nn[0]) continue;
          const long long id = gidx(g, ii, jj, kk);
          double us[3];
#pragma unroll
          for (int c = 0; c < 3; ++c)
            us[c] = predict_bc(g, L.f, ii, jj, kk, c, __ldg(L.u0 + c * np + id), __ldg(L.v0 + c * np + id),
                               __ldg(L.a0 + c * np + id), dt);
          if (ox == 0 && oy == 0 && oz == 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) own_us[c] = us[c];
          }
          const double* cb = coef + ((ox + 1) + 3 * ((oy + 1) + 3 * (oz + 1))) * 9;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int d = 0; d < 3; ++d) f[c] = fma(__ldg(cb + c * 3 + d), us[d], f[c]);
          }
        }
      }
    }
    const double mult = (cl[0] == 1 ? 2.0 : 1.0) * (cl[1] == 1 ? 2.0 : 1.0) * (cl[2] == 1 ? 2.0 : 1.0);
    const double inv_m = 1.0 / (L.mass_e * mult);
    const long long id = gidx(g, i, j, k);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double sv;
      const bool free_dof = dof_code(g, L.f, i, j, k, c, &sv) == DOF_FREE;
      double an = 0.0, vn = 0.0;
      if (free_dof) {
        an = -f[c] * inv_m;
        vn = fma(hdt, __ldg(L.a0 + c * np + id) + an, __ldg(L.v0 + c * np + id));
        if (L.with_norm) {
          const double up = L.u1[c * np + id], vp = L.v1[c * np + id];
          const double d = (own_us[c] - up) + dt * (vn - vp);
          const double w = own_us[c] + dt * vn;
          num = fma(d, d, num);
          den = fma(w, w, den);
        }
      }
      L.u1[c * np + id] = own_us[c];
      L.v1[c * np + id] = vn;
      L.a1[c * np + id] = an;
    }
  }
  block_partial<SURF_BLOCK>(num, den, L.partial, slot0 + blockIdx.x);
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

dim3 interior_grid(const Geom& g) {
  const long long ix = g.nn[0] - 2, iy = g.nn[1] - 2, iz = g.nn[2] - 2;
  if (ix <= 0 || iy <= 0 || iz <= 0) return dim3(0, 0, 0);
  return dim3(cdiv(ix, TX), cdiv(iy, TY), cdiv(iz, ZC));
}

}  // namespace

int fom_partial_slots(const Geom& g) {
  const dim3 gi = interior_grid(g);
  return (int)((long long)gi.x * gi.y * gi.z + cdiv(surface_count(g), SURF_BLOCK));
}

void launch_fom_advance(const FomLaunch& L, const InteriorStencil& st, cudaStream_t s, int* launches) {
  const dim3 gi = interior_grid(L.g);
  const int n_int = gi.x * gi.y * gi.z;
  if (n_int > 0) {
    fom_interior_kernel<<<gi, dim3(TX, TY), 0, s>>>(L, st);
    ++*launches;
  }
  const unsigned nb = cdiv(surface_count(L.g), SURF_BLOCK);
  fom_surface_kernel<<<nb, SURF_BLOCK, 0, s>>>(L, n_int);
  ++*launches;
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
