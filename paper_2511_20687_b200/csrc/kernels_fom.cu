// K1: fused FOM advance -- explicit Newmark (beta = 0, gamma = 1/2) step of a hex8
// linear-elastic box subdomain with lumped mass (A.1 P:L1934-1947),
// in the two-vector (u, w) form, w = v + dt/2 a (SURVEY 8(d) "leapfrog"; R30):
//
//   u* = u + dtp w            on free DOFs; 0 on Dirichlet DOFs; s on Schwarz DOFs
//   f  = K u*                 (matrix-free 27-point merged hex8 stencil, 153 nonzeros/node)
//   a' = -f / m_L ,  w' = w + cw a'  on free DOFs (w' = a' = 0 on constrained DOFs)
//   partial sums of  num = ||dt (w' - w_prev)/2||^2  and  den = ||u* + dt (w + cv a')||^2
//
// A Schwarz sweep uses dtp = cw = dt, cv = dt/2: then u* is the Newmark predictor
// u + dt v + dt^2/2 a, v' = w + dt/2 a' = v + dt/2 (a + a') and w' = v' + dt/2 a', and
// (u* - u*_prev) + dt (v' - v'_prev) = dt (w' - w'_prev)/2 on free DOFs because u* depends only
// on the checkpoint (eq:conv_criterion P:L443-467).  dtp = 0 with cw = (dt_new - dt_old)/2 changes
// the step a stored w refers to; cw = -dt/2 recovers v = w - dt/2 a for osam_get_state.
//
// Two kernels make one K1:
//   * the tiled kernel covers every node.  A block owns a TX x TY tile in (x, y) and a balanced
//     chunk of node planes in z; one thread streams the checkpoint planes (u, w; tile + one-node
//     halo) with 4D TMA loads into a 3-deep mbarrier ring.  Each staged plane is converted once to
//     u* in shared memory; each thread then loads its 3x3 in-plane neighbourhood once (27 shared
//     loads) and applies it to the forces of node planes m+1, m, m-1 held in registers (2.5D
//     streaming).  A warp is one x-row, so the (y, z) boundary class is warp-uniform: interior rows
//     use the 153-coefficient stencil from the kernel-parameter constant bank, face rows their class
//     table.  Lanes on an x-face write it only when the face is fully constrained (no force needed).
//   * the x-face kernel covers x-faces with free DOFs (a node per thread, class table).
// No atomics; every sum has a fixed order, so results are bitwise repeatable.
#include "osam_internal.h"

namespace osam {

namespace {

constexpr int TX = 32;
constexpr int TY = 8;
constexpr int NT = TX * TY;
constexpr int ZC = 16;  // target z-planes per block (balanced split)
constexpr int XF_BLOCK = 128;

__device__ __forceinline__ long long gidx(const Geom& g, int i, int j, int k) {
  return i + (long long)g.px * (j + (long long)g.nn[1] * k);
}

__device__ __forceinline__ int axis_class(int idx, int nn) { return idx == 0 ? 0 : (idx == nn - 1 ? 2 : 1); }

// Boundary data of a node on the surface: Dirichlet component mask and the Schwarz value
// (first Schwarz face, in face order, holding the node).  Dirichlet > Schwarz > free.
struct NodeBC {
  unsigned dmask;
  bool sw;
  double s[3];
};

__device__ __forceinline__ NodeBC node_bc(const Geom& g, const Faces& F, int i, int j, int k) {
  NodeBC b;
  b.dmask = 0;
  b.sw = false;
  b.s[0] = b.s[1] = b.s[2] = 0.0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const int v = ax == 0 ? i : (ax == 1 ? j : k);
    const bool on = v == ((f & 1) ? g.nn[ax] - 1 : 0);
    if (on) {
      b.dmask |= F.dir[f];
      if (F.sw[f] && !b.sw) {
        b.sw = true;
        // in-face index a + nn[o0] * b with (o0, o1) the two other axes in ascending order
        const long long fi = ax == 0 ? (j + (long long)g.nn[1] * k)
                                     : (ax == 1 ? (i + (long long)g.nn[0] * k) : (i + (long long)g.nn[0] * j));
        const long long nf = F.nface[f];
#pragma unroll
        for (int c = 0; c < 3; ++c) b.s[c] = F.s[f][c * nf + fi];
      }
    }
  }
  return b;
}

// Boundary info of a staged (x, y) position, fixed across z-planes: bits 0-2 Dirichlet mask of
// the x/y faces holding it, bits 3-5 the first Schwarz face among faces 0-3 (7: none), bit 6 set
// iff the position lies in the box.  PINFO_FREE = in the box and on no x/y face.
constexpr int PINFO_FREE = 64 | (7 << 3);

__device__ __forceinline__ int pos_info(const Geom& g, const Faces& F, int ii, int jj) {
  if (ii < 0 || ii > g.nn[0] - 1 || jj < 0 || jj > g.nn[1] - 1) return 0;
  unsigned dm = 0;
  int sf = 7;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int v = f < 2 ? ii : jj;
    const bool on = v == ((f & 1) ? g.nn[f >> 1] - 1 : 0);
    if (on) {
      dm |= F.dir[f];
      if (F.sw[f] && sf == 7) sf = f;
    }
  }
  return (int)dm | (sf << 3) | 64;
}

// Boundary overwrite of the predictor at a staged position off the z-faces, from its pos_info.
__device__ __forceinline__ void apply_bc_xy(const Geom& g, const Faces& F, int info, int ii, int jj, int m,
                                            double p[3]) {
  const int sf = (info >> 3) & 7;
  double sv[3] = {0.0, 0.0, 0.0};
  if (sf != 7) {
    const long long fi = sf < 2 ? (jj + (long long)g.nn[1] * m) : (ii + (long long)g.nn[0] * m);
    const double* sp = sf == 0 ? F.s[0] : (sf == 1 ? F.s[1] : (sf == 2 ? F.s[2] : F.s[3]));
    const long long nf = sf == 0 ? F.nface[0] : (sf == 1 ? F.nface[1] : (sf == 2 ? F.nface[2] : F.nface[3]));
#pragma unroll
    for (int c = 0; c < 3; ++c) sv[c] = sp[c * nf + fi];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = ((info >> c) & 1) ? 0.0 : (sf != 7 ? sv[c] : p[c]);
}

__device__ __forceinline__ bool is_boundary(const Geom& g, int i, int j, int k) {
  return i == 0 || j == 0 || k == 0 || i == g.nn[0] - 1 || j == g.nn[1] - 1 || k == g.nn[2] - 1;
}

// predictor with the boundary overwrite of a surface position
__device__ __forceinline__ void apply_bc(const Geom& g, const Faces& F, int i, int j, int k, double p[3]) {
  const NodeBC b = node_bc(g, F, i, j, k);
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = ((b.dmask >> c) & 1) ? 0.0 : (b.sw ? b.s[c] : p[c]);
}

// free-DOF mask (bit c) of a surface node
__device__ __forceinline__ unsigned free_mask(const Geom& g, const Faces& F, int i, int j, int k) {
  const NodeBC b = node_bc(g, F, i, j, k);
  return b.sw ? 0u : (~b.dmask) & 7u;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
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

// Staged x-range [x0, x0 + PX) with x0 = 32 bx - 2: the TMA box must start on a 16-byte
// boundary in the innermost dimension (an odd fp64 start coordinate raises an illegal
// instruction on sm_100a), so the left halo is two columns wide (the first is unused).
constexpr int PX = TX + 4;
constexpr int PY = TY + 2;
constexpr int PLANE = PX * PY;                             // positions per staged plane
constexpr int NSTAGE = 4;  // TMA ring: 2 planes in flight, the current one, the previous one (own w)
constexpr int NUST = 3;    // u* buffers: previous plane (own u* at finish), current, next
constexpr int ARR_BYTES = 3 * PLANE * 8;                   // one array (x,y,z comps) of one plane
constexpr int ARR_STRIDE = (ARR_BYTES + 127) / 128 * 128;  // 128-B aligned TMA destinations
constexpr int STAGE_BYTES = 2 * ARR_STRIDE;                // u, w
constexpr int SMEM_TILED = NSTAGE * STAGE_BYTES + NUST * ARR_STRIDE + 64;

// ---- interior rows: parity-reduced stencil ---------------------------------------------
// On a uniform box every interior block K_cd(ox, oy, oz) is even or odd in ox and in oy (the 1D
// factors M, S are symmetric, G, Gt antisymmetric): diagonal blocks even-even, xy/yx odd-odd,
// xz/zx odd-even, yz/zy even-odd (verified entry by entry on the host at create).  So the 3x3
// in-plane sum collapses onto 9 symmetric combinations P[xk][yk] of each component (xk, yk in
// {C: centre, E: pair sum, O: pair difference}), formed once per staged plane and applied to
// the three target planes with 14 (oz = 0) or 22 (oz = +-1) coefficients; the oz = +1 slice reuses
// the oz = -1 coefficients with the sign of the z-parity (odd for the xz, zx, yz, zy blocks).
enum { PC = 0, PE = 1, PO = 2 };

// the 9 combinations of one component around the thread's node (a = staged (-1,-1) neighbour)
__device__ __forceinline__ void combos(const double* a, double P[9]) {
  double cr[3], er[3], orr[3];
#pragma unroll
  for (int oy = 0; oy < 3; ++oy) {
    const double l = a[oy * PX], c = a[oy * PX + 1], r = a[oy * PX + 2];
    cr[oy] = c;
    er[oy] = l + r;
    orr[oy] = r - l;
  }
  P[PC * 3 + PC] = cr[1];
  P[PC * 3 + PE] = cr[0] + cr[2];
  P[PC * 3 + PO] = cr[2] - cr[0];
  P[PE * 3 + PC] = er[1];
  P[PE * 3 + PE] = er[0] + er[2];
  P[PE * 3 + PO] = er[2] - er[0];
  P[PO * 3 + PC] = orr[1];
  P[PO * 3 + PE] = orr[0] + orr[2];
  P[PO * 3 + PO] = orr[2] - orr[0];
}

// acc += sum_{ox,oy} K_cd(ox, oy, slice) w_d(ox, oy) for one block (c, d); ZNEG: use the oz = -1
// slice with the sign of the z-parity (the oz = +1 slice)
template <int SL, bool ZNEG, int c, int d>
__device__ __forceinline__ void contrib(double& acc, const double P[9], const InteriorStencil& S) {
  const double* k = S.k[SL][c][d];  // K00, K10, K01, K11
  constexpr bool zodd = (c == 2) != (d == 2);
  constexpr double sg = (ZNEG && zodd) ? -1.0 : 1.0;
  if (c == d) {
    acc = fma(sg * k[0], P[PC * 3 + PC], acc);
    acc = fma(sg * k[1], P[PE * 3 + PC], acc);
    acc = fma(sg * k[2], P[PC * 3 + PE], acc);
    acc = fma(sg * k[3], P[PE * 3 + PE], acc);
  } else if (c != 2 && d != 2) {  // xy, yx: odd-odd
    acc = fma(sg * k[3], P[PO * 3 + PO], acc);
  } else if (SL != 1) {
    if (c == 0 || d == 0) {  // xz, zx: odd in x, even in y
      acc = fma(sg * k[1], P[PO * 3 + PC], acc);
      acc = fma(sg * k[3], P[PO * 3 + PE], acc);
    } else {  // yz, zy: even in x, odd in y
      acc = fma(sg * k[2], P[PC * 3 + PO], acc);
      acc = fma(sg * k[3], P[PE * 3 + PO], acc);
    }
  }
}

template <int d, bool DA, bool DB, bool DC>
__device__ __forceinline__ void fast_comp(double A[3], double B[3], double C[3], const double* us, int base,
                                          const InteriorStencil& S) {
  double P[9];
  combos(us + d * PLANE + base, P);
  if (DA) {
    contrib<0, false, 0, d>(A[0], P, S);
    contrib<0, false, 1, d>(A[1], P, S);
    contrib<0, false, 2, d>(A[2], P, S);
  }
  if (DB) {
    contrib<1, false, 0, d>(B[0], P, S);
    contrib<1, false, 1, d>(B[1], P, S);
    contrib<1, false, 2, d>(B[2], P, S);
  }
  if (DC) {
    contrib<0, true, 0, d>(C[0], P, S);
    contrib<0, true, 1, d>(C[1], P, S);
    contrib<0, true, 2, d>(C[2], P, S);
  }
}

// interior rows: the staged plane's contributions to the targets that are needed
// (A: node plane m+1 sees plane m at oz = -1; B: plane m, oz = 0; C: plane m-1, oz = +1)
template <bool DA, bool DB, bool DC>
__device__ __forceinline__ void plane_fast(double A[3], double B[3], double C[3], const double* us, int base,
                                           const InteriorStencil& S) {
  fast_comp<0, DA, DB, DC>(A, B, C, us, base, S);
  fast_comp<1, DA, DB, DC>(A, B, C, us, base, S);
  fast_comp<2, DA, DB, DC>(A, B, C, us, base, S);
}

// Face rows / face planes: full 3x3 blocks from the class table (L1 broadcast).
template <int OZ>
__device__ __forceinline__ void plane_class(double acc[3], const double* us, int base,
                                            const double* __restrict__ cls_coef) {
#pragma unroll
  for (int oy = 0; oy < 3; ++oy) {
#pragma unroll
    for (int ox = 0; ox < 3; ++ox) {
      const int q = base + oy * PX + ox;
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
__device__ __forceinline__ void target_any(double acc[3], const double* us, int base, int cy, int cz,
                                           const InteriorStencil& S, const double* coef) {
  if (cy == 1 && cz == 1) {
    double d0[3] = {0.0, 0.0, 0.0}, d1[3] = {0.0, 0.0, 0.0};
    if (OZ == 0) plane_fast<true, false, false>(acc, d0, d1, us, base, S);
    if (OZ == 1) plane_fast<false, true, false>(d0, acc, d1, us, base, S);
    if (OZ == 2) plane_fast<false, false, true>(d0, d1, acc, us, base, S);
  } else {
    plane_class<OZ>(acc, us, base, coef + (size_t)(1 + 3 * (cy + 3 * cz)) * 27 * 9);
  }
}

// Face rows / face planes (rare): the three targets' contributions of one staged plane from the
// class tables, out of line to keep the hot loop small.
struct Contrib3 {
  double v[9];
};

__device__ __noinline__ Contrib3 plane_slow(const double* us, int base, int cy, int czA, int czB, int czC,
                                             const InteriorStencil& S, const double* coef) {
  Contrib3 r;
  double A[3] = {0.0, 0.0, 0.0}, B[3] = {0.0, 0.0, 0.0}, C[3] = {0.0, 0.0, 0.0};
  target_any<0>(A, us, base, cy, czA, S, coef);
  target_any<1>(B, us, base, cy, czB, S, coef);
  target_any<2>(C, us, base, cy, czC, S, coef);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r.v[c] = A[c];
    r.v[3 + c] = B[c];
    r.v[6 + c] = C[c];
  }
  return r;
}

__device__ __noinline__ void apply_bc_full(const Geom& g, const Faces& F, int i, int j, int k, double& p0, double& p1,
                                           double& p2) {
  double p[3] = {p0, p1, p2};
  apply_bc(g, F, i, j, k, p);
  p0 = p[0];
  p1 = p[1];
  p2 = p[2];
}

// Per-thread constants of the tiled kernel.
struct Tile {
  int t, qo, base, q1;
  bool has1;
  int info0, info1;
  int x0, y0, i, j;
  bool active, xface, writer;
  int cy, kbeg, kend, nplanes;
  long long id0;
};

// One staged plane (iteration it, staged plane m = kbeg - 1 + it).  Accumulator slots rotate by
// role: A = acc[SA] (node plane m+1), B = acc[SB] (plane m), C = acc[SC] (plane m-1, finished
// here if it lies in [kbeg, kend], then zeroed to become the next A).  Targets outside the chunk
// are accumulated too (and never used): that keeps every iteration identical.
template <int SA, int SB, int SC>
__device__ __forceinline__ void k1_iter(const FomLaunch& L, const InteriorStencil& S, const Tile& T, int it,
                                        double (&acc)[3][3], double& num, double& den, double* raw, double* ust,
                                        unsigned long long* bar, const CUtensorMap* tu, const CUtensorMap* tw) {
  constexpr int U3 = (3 - SA) % 3;  // == it % 3
  const Geom& g = L.g;
  const int nz = g.nn[2] - 1;
  const long long np = g.npad;
  const int m = T.kbeg - 1 + it;
  const int kf = m - 1;
  const bool fin = T.writer && kf >= T.kbeg && kf <= T.kend;
  const long long id = T.id0 + (long long)kf * g.plane;
  double qw[3] = {0.0, 0.0, 0.0};
  if (fin && L.with_norm && !T.xface) {  // previous Schwarz iterate (norm), issued before the wait
#pragma unroll
    for (int c = 0; c < 3; ++c) qw[c] = L.w1[c * np + id];
  }
  const int s = it & (NSTAGE - 1);
  mbar_wait(&bar[s], (unsigned)((it / NSTAGE) & 1));
  const double* ru = raw + (size_t)s * (STAGE_BYTES / 8);
  const double* rw = ru + ARR_STRIDE / 8;
  double* us = ust + U3 * (ARR_STRIDE / 8);
  // predictor u* = u + dtp w (TMA zero-fills out-of-box positions; the padding columns hold 0)
  {
    const bool mval = m >= 0 && m <= nz;
    const bool bplane = (m == 0) || (m == nz);
    const double dtp = L.dtp;
    double p[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) p[c] = fma(dtp, rw[c * PLANE + T.t], ru[c * PLANE + T.t]);
    if (mval && T.info0 != PINFO_FREE && T.info0 != 0) {
      if (bplane)
        apply_bc_full(g, L.f, T.x0 + T.t % PX, T.y0 + T.t / PX, m, p[0], p[1], p[2]);
      else
        apply_bc_xy(g, L.f, T.info0, T.x0 + T.t % PX, T.y0 + T.t / PX, m, p);
    } else if (bplane && T.info0 == PINFO_FREE) {
      apply_bc(g, L.f, T.x0 + T.t % PX, T.y0 + T.t / PX, m, p);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) us[c * PLANE + T.t] = p[c];
    if (T.has1) {
      const int q1 = T.q1;
#pragma unroll
      for (int c = 0; c < 3; ++c) p[c] = fma(dtp, rw[c * PLANE + q1], ru[c * PLANE + q1]);
      if (mval && T.info1 != PINFO_FREE && T.info1 != 0) {
        if (bplane)
          apply_bc_full(g, L.f, T.x0 + q1 % PX, T.y0 + q1 / PX, m, p[0], p[1], p[2]);
        else
          apply_bc_xy(g, L.f, T.info1, T.x0 + q1 % PX, T.y0 + q1 / PX, m, p);
      } else if (bplane && T.info1 == PINFO_FREE) {
        apply_bc_full(g, L.f, T.x0 + q1 % PX, T.y0 + q1 / PX, m, p[0], p[1], p[2]);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) us[c * PLANE + q1] = p[c];
    }
  }
  __syncthreads();
  if (T.t == 0 && it + 2 < T.nplanes) {  // refill: stage (it+2) % 4 was last read in iteration it-1
    const int s2 = (it + 2) & (NSTAGE - 1);
    double* dst = raw + (size_t)s2 * (STAGE_BYTES / 8);
    mbar_expect_tx(&bar[s2], 2 * ARR_BYTES);
    tma_load_4d(dst, tu, T.x0, T.y0, m + 2, 0, &bar[s2]);
    tma_load_4d(dst + ARR_STRIDE / 8, tw, T.x0, T.y0, m + 2, 0, &bar[s2]);
  }
  if (T.active) {
    double* A = acc[SA];
    double* B = acc[SB];
    double* C = acc[SC];
    if (T.cy == 1 && m >= 2 && m <= nz - 2) {
      plane_fast<true, true, true>(A, B, C, us, T.base, S);
    } else {
      const Contrib3 r = plane_slow(us, T.base, T.cy, axis_class(m + 1, g.nn[2]), axis_class(m, g.nn[2]),
                                    axis_class(kf, g.nn[2]), S, L.coef);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        A[c] += r.v[c];
        B[c] += r.v[3 + c];
        C[c] += r.v[6 + c];
      }
    }
    if (fin) {
      // own u* and checkpoint w of plane kf = m-1, kept in shared memory since iteration it-1
      const double* pus = ust + ((U3 + 2) % 3) * (ARR_STRIDE / 8) + T.qo;
      const double* pws = raw + (size_t)((it - 1) & (NSTAGE - 1)) * (STAGE_BYTES / 8) + ARR_STRIDE / 8 + T.qo;
      double* u1 = L.u1 + id;
      double* w1 = L.w1 + id;
      const int cz = axis_class(kf, g.nn[2]);
      if (T.xface) {  // fully constrained x-face node: prescribed u, w = a = 0
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          u1[c * np] = pus[c * PLANE];
          w1[c * np] = 0.0;
          if (L.a_out) L.a_out[c * np + id] = 0.0;
        }
      } else if (T.cy == 1 && cz == 1 && L.a_out == nullptr) {  // interior node, all DOFs free
        const double inv_m = L.inv_mass[7];
        double pu[3], an[3], wn[3], pw[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pu[c] = pus[c * PLANE];
          pw[c] = pws[c * PLANE];
          an[c] = -C[c] * inv_m;
          wn[c] = fma(L.cw, an[c], pw[c]);
          u1[c * np] = pu[c];
          w1[c * np] = wn[c];
        }
        if (L.with_norm) {
          const double hdt = 0.5 * L.dt;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double d = hdt * (wn[c] - qw[c]);
            const double w = fma(L.dt, fma(L.cv, an[c], pw[c]), pu[c]);
            num = fma(d, d, num);
            den = fma(w, w, den);
          }
        }
      } else {
        const unsigned fm = (T.cy != 1 || cz != 1) ? free_mask(g, L.f, T.i, T.j, kf) : 7u;
        const double inv_m = L.inv_mass[1 + 2 * (T.cy == 1) + 4 * (cz == 1)];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double pu = pus[c * PLANE], pw = pws[c * PLANE];
          double an = 0.0, wn = 0.0;
          if ((fm >> c) & 1) {
            an = -C[c] * inv_m;
            wn = fma(L.cw, an, pw);
            if (L.with_norm) {
              const double d = 0.5 * L.dt * (wn - qw[c]);
              const double w = fma(L.dt, fma(L.cv, an, pw), pu);
              num = fma(d, d, num);
              den = fma(w, w, den);
            }
          }
          u1[c * np] = pu;
          w1[c * np] = wn;
          if (L.a_out) L.a_out[c * np + id] = an;
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) acc[SC][c] = 0.0;
}

__global__ void __launch_bounds__(NT, 2)
    fom_tiled_kernel(const __grid_constant__ FomLaunch L, const __grid_constant__ InteriorStencil S,
                     const __grid_constant__ CUtensorMap tu, const __grid_constant__ CUtensorMap tw) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* raw = reinterpret_cast<double*>(smem);
  double* ust = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + NSTAGE * STAGE_BYTES + NUST * ARR_STRIDE);
  const Geom& g = L.g;
  const int nx = g.nn[0] - 1, ny = g.nn[1] - 1;
  Tile T;
  const int tx = threadIdx.x, ty = threadIdx.y;
  T.t = ty * TX + tx;
  T.x0 = blockIdx.x * TX - 2;  // node coordinates of staged position (0,0)
  T.y0 = blockIdx.y * TY - 1;
  T.i = T.x0 + 2 + tx;
  T.j = T.y0 + 1 + ty;
  T.active = (T.i <= nx) && (T.j <= ny);
  T.xface = (T.i == 0) || (T.i == nx);
  const int xs = T.i == 0 ? 0 : 1;
  const bool xf_full = T.xface && (L.f.dir[xs] == 7 || L.f.sw[xs]);
  T.writer = T.active && (!T.xface || xf_full);
  T.cy = axis_class(T.j, g.nn[1]);  // warp-uniform (a warp is one x-row)
  T.kbeg = (int)((long long)blockIdx.z * g.nn[2] / gridDim.z);
  T.kend = (int)((long long)(blockIdx.z + 1) * g.nn[2] / gridDim.z) - 1;
  T.nplanes = T.kend - T.kbeg + 3;
  T.qo = (ty + 1) * PX + (tx + 2);
  T.base = ty * PX + tx + 1;
  T.q1 = T.t + NT;
  T.has1 = T.q1 < PLANE;
  T.info0 = pos_info(g, L.f, T.x0 + T.t % PX, T.y0 + T.t / PX);
  T.info1 = T.has1 ? pos_info(g, L.f, T.x0 + T.q1 % PX, T.y0 + T.q1 / PX) : 0;
  T.id0 = T.i + (long long)g.px * T.j;

  if (T.t == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (T.t == 0) {
    for (int it = 0; it < 2 && it < T.nplanes; ++it) {
      double* dst = raw + (size_t)it * (STAGE_BYTES / 8);
      mbar_expect_tx(&bar[it], 2 * ARR_BYTES);
      tma_load_4d(dst, &tu, T.x0, T.y0, T.kbeg - 1 + it, 0, &bar[it]);
      tma_load_4d(dst + ARR_STRIDE / 8, &tw, T.x0, T.y0, T.kbeg - 1 + it, 0, &bar[it]);
    }
  }

  double acc[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  double num = 0.0, den = 0.0;
  for (int it = 0; it < T.nplanes;) {  // unrolled by the period 3 of the slot rotation
    k1_iter<0, 1, 2>(L, S, T, it, acc, num, den, raw, ust, bar, &tu, &tw);
    if (++it >= T.nplanes) break;
    k1_iter<2, 0, 1>(L, S, T, it, acc, num, den, raw, ust, bar, &tu, &tw);
    if (++it >= T.nplanes) break;
    k1_iter<1, 2, 0>(L, S, T, it, acc, num, den, raw, ust, bar, &tu, &tw);
    ++it;
  }
  const int slot = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  block_partial<NT>(num, den, L.partial, slot);
}

// Nodes on an x-face with free DOFs (one per thread): gather over the 18 neighbours inside the
// box, class-table stencil.  side_mask bit 0: face x = 0, bit 1: face x = nx.
__global__ void __launch_bounds__(XF_BLOCK) fom_xface_kernel(const FomLaunch L, int slot0, int side_mask) {
  const Geom& g = L.g;
  const long long np = g.npad;
  const long long nf = (long long)g.nn[1] * g.nn[2];
  const int nsides = (side_mask & 1) + ((side_mask >> 1) & 1);
  const long long t = blockIdx.x * (long long)XF_BLOCK + threadIdx.x;
  const double dtp = L.dtp;
  const int nx = g.nn[0] - 1;
  double num = 0.0, den = 0.0;
  if (t < nsides * nf) {
    const int side = (side_mask == 2) ? 1 : (t >= nf ? 1 : 0);
    const long long r = t - (t >= nf ? nf : 0);
    const int i = side ? nx : 0;
    const int j = (int)(r % g.nn[1]);
    const int k = (int)(r / g.nn[1]);
    const long long id = gidx(g, i, j, k);
    const unsigned fm = free_mask(g, L.f, i, j, k);
    double own[3] = {0.0, 0.0, 0.0};
    double f[3] = {0.0, 0.0, 0.0};
    const int cl = (side ? 2 : 0) + 3 * (axis_class(j, g.nn[1]) + 3 * axis_class(k, g.nn[2]));
    const double* coef = L.coef + (size_t)cl * 27 * 9;
    const int oxlo = side ? -1 : 0;
    for (int oz = -1; oz <= 1; ++oz) {
      const int kk = k + oz;
      if (kk < 0 || kk > g.nn[2] - 1) continue;
      for (int oy = -1; oy <= 1; ++oy) {
        const int jj = j + oy;
        if (jj < 0 || jj > g.nn[1] - 1) continue;
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int ox = oxlo + dx;
          const int ii = i + ox;
          const long long q = gidx(g, ii, jj, kk);
          double p[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) p[c] = fma(dtp, __ldg(L.w0 + c * np + q), __ldg(L.u0 + c * np + q));
          if (is_boundary(g, ii, jj, kk)) apply_bc(g, L.f, ii, jj, kk, p);
          if (ox == 0 && oy == 0 && oz == 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) own[c] = p[c];
          }
          const double* cb = coef + ((ox + 1) + 3 * ((oy + 1) + 3 * (oz + 1))) * 9;
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) f[c] = fma(__ldg(cb + c * 3 + d), p[d], f[c]);
        }
      }
    }
    const double inv_m = L.inv_mass[(axis_class(j, g.nn[1]) == 1 ? 2 : 0) + (axis_class(k, g.nn[2]) == 1 ? 4 : 0)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double an = 0.0, wn = 0.0;
      if ((fm >> c) & 1) {
        const double w0 = __ldg(L.w0 + c * np + id);
        an = -f[c] * inv_m;
        wn = fma(L.cw, an, w0);
        if (L.with_norm) {
          const double d = 0.5 * L.dt * (wn - L.w1[c * np + id]);
          const double v = fma(L.cv, an, w0);
          const double w = fma(L.dt, v, own[c]);
          num = fma(d, d, num);
          den = fma(w, w, den);
        }
      }
      L.u1[c * np + id] = own[c];
      L.w1[c * np + id] = wn;
      if (L.a_out) L.a_out[c * np + id] = an;
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
  const long long inner = (n2 > 2 ? n2 - 2 : 0);
  return 2 * n0 * n1 + 2 * n0 * inner + 2 * (n1 > 2 ? n1 - 2 : 0) * inner;
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
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    if (!F.sw[f] || t >= F.nface[f]) continue;
    const int ax = f >> 1;
    const int side = (f & 1) ? g.nn[ax] - 1 : 0;
    int i, j, k;
    if (ax == 0) {
      i = side;
      j = (int)(t % g.nn[1]);
      k = (int)(t / g.nn[1]);
    } else if (ax == 1) {
      j = side;
      i = (int)(t % g.nn[0]);
      k = (int)(t / g.nn[0]);
    } else {
      k = side;
      i = (int)(t % g.nn[0]);
      j = (int)(t / g.nn[0]);
    }
    const long long q = gidx(g, i, j, k);
    for (int c = 0; c < 3; ++c) F.s[f][c * (long long)F.nface[f] + t] = u[c * g.npad + q];
  }
}

// Dirichlet u := 0 (if zero_u), constrained w := 0 on every surface node.
__global__ void zero_constrained_kernel(Geom g, Faces F, double* u, double* w, int zero_u) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= surface_count(g)) return;
  int i, j, k;
  surface_node(g, t, &i, &j, &k);
  const long long q = gidx(g, i, j, k);
  const NodeBC b = node_bc(g, F, i, j, k);
  for (int c = 0; c < 3; ++c) {
    const bool dir = (b.dmask >> c) & 1;
    if (dir || b.sw) {
      w[c * g.npad + q] = 0.0;
      if (zero_u && dir) u[c * g.npad + q] = 0.0;
    }
  }
}

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

dim3 tiled_grid(const Geom& g) { return dim3(cdiv(g.nn[0], TX), cdiv(g.nn[1], TY), cdiv(g.nn[2], ZC)); }

int xface_sides(const Faces& f) {
  int m = 0;
  for (int s = 0; s < 2; ++s)
    if (!(f.dir[s] == 7 || f.sw[s])) m |= 1 << s;
  return m;
}

unsigned xface_blocks(const Geom& g, const Faces& f) {
  const int m = xface_sides(f);
  const int ns = (m & 1) + ((m >> 1) & 1);
  return ns ? cdiv((long long)ns * g.nn[1] * g.nn[2], XF_BLOCK) : 0u;
}

}  // namespace

int fom_partial_slots(const Geom& g, const Faces& f) {
  const dim3 gi = tiled_grid(g);
  return (int)((long long)gi.x * gi.y * gi.z + xface_blocks(g, f));
}

void launch_fom_advance(const FomLaunch& L, const InteriorStencil& st, const CUtensorMap* tm, cudaStream_t s,
                        int* launches) {
  const dim3 gi = tiled_grid(L.g);
  const int n_int = gi.x * gi.y * gi.z;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(fom_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TILED);
    attr_set = true;
  }
  fom_tiled_kernel<<<gi, dim3(TX, TY), SMEM_TILED, s>>>(L, st, tm[0], tm[1]);
  debug_check("fom_tiled_kernel", s);
  ++*launches;
  const unsigned xb = xface_blocks(L.g, L.f);
  if (xb > 0) {
    fom_xface_kernel<<<xb, XF_BLOCK, 0, s>>>(L, n_int, xface_sides(L.f));
    debug_check("fom_xface_kernel", s);
    ++*launches;
  }
}

int make_state_tmaps(const Geom& g, double* const arrays[2], CUtensorMap out[2]) {
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
  for (int q = 0; q < 2; ++q) {
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
  face_gather_kernel<<<cdiv(nmax, 256), 256, 0, s>>>(g, f, u);
  debug_check("face_gather_kernel", s);
}

void launch_fom_pack(const Geom& g, const double* src, double* dst, long long n, cudaStream_t s) {
  pack_kernel<<<cdiv(n, 256), 256, 0, s>>>(g, src, dst, n);
  debug_check("pack_kernel", s);
}

void launch_fom_unpack(const Geom& g, const double* src, double* dst, long long n, cudaStream_t s) {
  unpack_kernel<<<cdiv(n, 256), 256, 0, s>>>(g, src, dst, n);
  debug_check("unpack_kernel", s);
}

void launch_fom_zero_constrained(const Geom& g, const Faces& f, double* u, double* w, int zero_u, cudaStream_t s) {
  zero_constrained_kernel<<<cdiv(surface_count(g), 256), 256, 0, s>>>(g, f, u, w, zero_u);
  debug_check("zero_constrained_kernel", s);
}

}  // namespace osam
