// K1 tiled kernel for one tile shape K1_TX x K1_TY (included by kernels_fom.cu once per shape, each time
// inside its own namespace; no include guard on purpose).  Everything here depends on the tile shape:
// the staged-plane layout, the stencil's shared-memory offsets, the tile grid, the x-face CTAs, the TMA
// boxes and the launch.  See the header of kernels_fom.cu for the design.

constexpr int TX = K1_TX;  // tile width in x (a multiple of 16: even TMA start coordinates, whole sectors)
constexpr int TY = K1_TY;
constexpr int NT = TX * TY;
constexpr int NWARP = NT / 32;
constexpr int ZC = K1_ZC;  // target z-planes per block (balanced split)
constexpr int XF_BLOCK = NT;  // x-face work runs in extra CTAs of the tiled kernel (same block)
#ifndef OSAM_K1_PW
#define OSAM_K1_PW 0
#endif
// OSAM_K1_PW = 1: a dedicated producer warp (one more warp per CTA, the rows threadIdx.y >= TY) issues every TMA
// load, so no consumer warp carries the ~400 cycles of issue per plane and the CTA no longer runs at warp 0's pace.
constexpr int PW = (OSAM_K1_PW && 32 % K1_TX == 0) ? 1 : 0;
constexpr int NTB = NT + 32 * PW;                    // threads per CTA
constexpr int BY = TY + PW * (32 / (K1_TX > 32 ? 32 : K1_TX));  // blockDim.y

// Staged x-range [x0, x0 + PX) with x0 = 32 bx - 2: the TMA box must start on a 16-byte
// boundary in the innermost dimension (an odd fp64 start coordinate raises an illegal
// instruction on sm_100a), so the left halo is two columns wide (the first is unused).
constexpr int PX = TX + 4;
#ifndef OSAM_K1_WARP
#define OSAM_K1_WARP 0
#endif
// OSAM_K1_WARP = 1: every warp streams its own rows (its own TMA boxes, ring and full barriers; no empty
// barriers), so no warp waits for another; the staged box is the warp's WR rows plus the y halo.
constexpr int WR = 32 / TX;                          // node rows per warp
constexpr int SR = OSAM_K1_WARP ? WR : TY;           // node rows of one staged box
constexpr int NRING = OSAM_K1_WARP ? NWARP : 1;      // rings per CTA
constexpr int PY = SR + 2;
constexpr int PLANE = PX * PY;                             // positions per staged plane
#ifndef OSAM_NSTAGE
#define OSAM_NSTAGE 4
#endif
constexpr int NSTAGE = OSAM_NSTAGE;  // ring: NSTAGE-2 planes in flight, current, previous
constexpr int ARR_BYTES = 3 * PLANE * 8;                   // X (x,y,z comps) of one plane, with halo
constexpr int ARR_STRIDE = (ARR_BYTES + 127) / 128 * 128;  // 128-B aligned TMA destinations
constexpr int WPL = TX * SR;                               // staged positions of W (no halo)
constexpr int W_BYTES = 3 * WPL * 8;
constexpr int STAGE_BYTES = ARR_STRIDE + 2 * W_BYTES;  // X, W, W'_prev
constexpr int SMEM_TILED = NRING * NSTAGE * STAGE_BYTES + NRING * 2 * NSTAGE * 8;  // rings, barriers

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
__device__ __forceinline__ void fast_comp(double A[3], double B[3], double C[3], const double* xs, int base,
                                          const InteriorStencil& S) {
  double P[9];
  combos(xs + d * PLANE + base, P);
  if (DA) {
    contrib<0, false, 0, d>(A[0], P, S);
    contrib<0, false, 1, d>(A[1], P, S);
    contrib<0, false, 2, d>(A[2], P, S);
  }
  if (DC) {
    contrib<0, true, 0, d>(C[0], P, S);
    contrib<0, true, 1, d>(C[1], P, S);
    contrib<0, true, 2, d>(C[2], P, S);
  }
  if (DB) {
    contrib<1, false, 0, d>(B[0], P, S);
    contrib<1, false, 1, d>(B[1], P, S);
    contrib<1, false, 2, d>(B[2], P, S);
  }
}

// interior rows: the staged plane's contributions to the targets
// (A: node plane m+1 sees plane m at oz = -1; B: plane m, oz = 0; C: plane m-1, oz = +1)
template <bool DA, bool DB, bool DC>
__device__ __forceinline__ void plane_fast(double A[3], double B[3], double C[3], const double* xs, int base,
                                           const InteriorStencil& S) {
  fast_comp<0, DA, DB, DC>(A, B, C, xs, base, S);
  fast_comp<1, DA, DB, DC>(A, B, C, xs, base, S);
  fast_comp<2, DA, DB, DC>(A, B, C, xs, base, S);
}

// Face rows / face planes (rare): "row form" of the stencil, valid for every (y, z) class because
// the x-parity of each block holds for all lanes of the tiled kernel (x-face lanes never use the
// force): sum_ox K(ox, oy) w(ox, oy) = K(0, oy) c_row + K(1, oy) e_row (x-even blocks) or
// K(1, oy) o_row (x-odd blocks).  rowc holds {K(0, oy), K(1, oy)} per (cy, cz, slice, c, d, oy),
// built and checked on the host; out of line to keep the hot loop small.
struct Contrib3 {
  double v[9];
};

__device__ __noinline__ Contrib3 plane_slow(const double* xs, int base, int cy, int czA, int czB, int czC,
                                             const double* __restrict__ rowc) {
  const double* kt[3] = {rowc + ((cy * 3 + czA) * 3 + 0) * 54, rowc + ((cy * 3 + czB) * 3 + 1) * 54,
                         rowc + ((cy * 3 + czC) * 3 + 2) * 54};
  double acc[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double* a = xs + d * PLANE + base;
    double cr[3], er[3], orr[3];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) {
      const double l = a[oy * PX], c = a[oy * PX + 1], r = a[oy * PX + 2];
      cr[oy] = c;
      er[oy] = l + r;
      orr[oy] = r - l;
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const bool even = (c == 0) == (d == 0);
#pragma unroll
        for (int oy = 0; oy < 3; ++oy) {
          const double* k = kt[t] + ((c * 3 + d) * 3 + oy) * 2;
          if (even) {
            acc[t][c] = fma(__ldg(k), cr[oy], acc[t][c]);
            acc[t][c] = fma(__ldg(k + 1), er[oy], acc[t][c]);
          } else {
            acc[t][c] = fma(__ldg(k + 1), orr[oy], acc[t][c]);
          }
        }
      }
    }
  }
  Contrib3 r;
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int c = 0; c < 3; ++c) r.v[3 * t + c] = acc[t][c];
  return r;
}

// Tiles of the persistent tiled kernel: TX x TY nodes in (x, y), a balanced chunk of ~ZC node
// planes in z; tile t -> (bx, by, bz) with bx fastest.
struct TileGrid {
  int tx, ty, tz;
  __device__ __forceinline__ int count() const { return tx * ty * tz; }
};

// x-faces whose nodes have free DOFs (bit 0: x = 0, bit 1: x = nx): their forces come from xface_body
__host__ __device__ __forceinline__ int xface_sides(const Faces& f) {
  int m = 0;
  for (int s = 0; s < 2; ++s)
    if (!(f.dir[s] == 7 || f.sw[s])) m |= 1 << s;
  return m;
}

// x-tile columns: when the last node column x = nx sits alone in a tile (nx a multiple of TX) and the
// x+ face is fully constrained (Dirichlet in every component, or Schwarz), that column only copies
// its prescribed values (Q' = X, W' = a = 0): it is left out of the tiled grid and handled by
// xlast_copy_kernel (c4's 257^3 FOM: 8 instead of 9 columns).
__host__ __device__ __forceinline__ bool xlast_excluded(const Geom& g, const Faces& f) {
  const int nx = g.nn[0] - 1;
  return nx > 0 && nx % TX == 0 && (f.dir[1] == 7 || f.sw[1]);
}

__host__ __device__ __forceinline__ int tile_cols(const Geom& g, const Faces& f) {
  return xlast_excluded(g, f) ? (g.nn[0] - 1) / TX : (g.nn[0] + TX - 1) / TX;
}

__device__ __forceinline__ TileGrid tile_grid(const Geom& g, const Faces& f) {
  return TileGrid{tile_cols(g, f), (g.nn[1] + TY - 1) / TY, (g.nn[2] + ZC - 1) / ZC};
}

// Geometry of one tile as the producer and the consumers see it.
struct TileGeo {
  int x0, y0;        // node coordinates of staged position (0, 0)
  int kbeg, kend;    // node planes finished by this tile
  int nplanes;       // staged planes kbeg-1 .. kend+1
};

// First node plane of z-chunk b of tz.  CTAs are dispatched chunk layer by chunk layer (bz slowest), so the chunks
// taper: their sizes fall linearly from (1 + p/100) to (1 - p/100) of the mean, the long CTAs start first and the
// launch drains through short ones (the tail of a launch is one CTA duration at falling occupancy).  The number of
// chunks, and with it the halo planes re-read, is unchanged.  p = OSAM_ZTAPER (0: balanced split).  Measured
// (profiles/r7c_ab_k1_ztaper.log): K1 alone 0.178 -> 0.164 ms per launch (c3), the concurrent c3 step 946 -> 976
// steps/s at p = 55 (25: 964, 40: 972, 70: 968, 85: 952).
#ifndef OSAM_ZTAPER
#define OSAM_ZTAPER 55
#endif
__device__ __forceinline__ int zsplit(int nz, int tz, int b) {
  constexpr long long p = OSAM_ZTAPER;
  if (p == 0 || tz < 2) return (int)((long long)b * nz / tz);
  const long long c = (long long)b * (100 + p) * (tz - 1) - p * (long long)b * (b - 1);
  return (int)((long long)nz * c / (100LL * tz * (tz - 1)));
}

__device__ __forceinline__ TileGeo tile_geo(const Geom& g, const TileGrid& G, int t) {
  const int bx = t % G.tx, by = (t / G.tx) % G.ty, bz = t / (G.tx * G.ty);
  TileGeo o;
  o.x0 = bx * TX - 2;
  o.y0 = by * TY - 1;
  o.kbeg = zsplit(g.nn[2], G.tz, bz);
  o.kend = zsplit(g.nn[2], G.tz, bz + 1) - 1;
  o.nplanes = o.kend - o.kbeg + 3;
  return o;
}

// Per-thread constants of the current tile (kept small: every register counts for occupancy).
struct Tile {
  int i, j;
  int kbeg, kend, nplanes;
  unsigned flags;  // bit 0 active, bit 1 x-face lane, bit 2 writer, bits 3-4 cy (class of row j),
                   // bit 5 the tile reads the previous iterate (norm numerator, see needs_prev)
  long long id0;   // node index of (i, j, 0)
  __device__ __forceinline__ bool active() const { return flags & 1u; }
  __device__ __forceinline__ bool xface() const { return flags & 2u; }
  __device__ __forceinline__ bool writer() const { return flags & 4u; }
  __device__ __forceinline__ int cy() const { return (int)((flags >> 3) & 3u); }
  __device__ __forceinline__ bool prev() const { return flags & 32u; }
};

// staged positions of this thread: own node, (-1,-1) neighbour, W tile position
__device__ __forceinline__ int srow() { return OSAM_K1_WARP ? (int)threadIdx.y % WR : (int)threadIdx.y; }
__device__ __forceinline__ int pos_own() { return (srow() + 1) * PX + ((int)threadIdx.x + 2); }
__device__ __forceinline__ int pos_base() { return srow() * PX + (int)threadIdx.x + 1; }
__device__ __forceinline__ int pos_w() { return srow() * TX + (int)threadIdx.x; }

struct Maps {
  const CUtensorMap *x, *w, *wp;
};

// Does this tile read the previous iterate (W'_prev, or z_prev) for the convergence numerator?
// Within a controller step the stencil input u* = X changes between Schwarz iterations only at
// Schwarz DOFs (the predictor and the Dirichlet values are fixed, R30), so a node farther than one
// layer from every Schwarz face gets a bitwise identical a' and w' in every iteration and its
// numerator term is exactly 0: only tiles holding a node within one layer of a Schwarz face need it
// (R38).  Multi-substep intervals (z-form, z_out set) change u everywhere: always.
__device__ __forceinline__ bool needs_prev(const FomLaunch& L, const TileGeo& P) {
  if (!L.with_norm) return false;
  if (L.z_out) return true;
  const Geom& g = L.g;
  const int lo[3] = {P.x0 + 2, P.y0 + 1, P.kbeg};
  const int hi[3] = {min(P.x0 + 1 + TX, g.nn[0] - 1), min(P.y0 + TY, g.nn[1] - 1), P.kend};
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    if (L.f.sw[f] && ((f & 1) ? hi[ax] >= g.nn[ax] - 2 : lo[ax] <= 1)) return true;
  }
  return false;
}

// ---- the transfer in the K1 grid -------------------------------------------------
// Tile columns whose staged X box [bx TX - 2, bx TX + TX + 1] holds a node of a Schwarz x-face: lo columns at
// x = 0 (only column 0: column 1 starts at TX - 2 > 0), hi columns at x = nx.  These tiles are dispatched last and
// wait for the transfer CTAs; every other tile reads no Schwarz value.
__host__ __device__ __forceinline__ void wait_cols(const Geom& g, const Faces& f, int tx, int& lo, int& hi) {
  const int nx = g.nn[0] - 1;
  lo = f.sw[0] ? 1 : 0;
  hi = 0;
  if (f.sw[1])
    for (int bx = tx - 1; bx >= lo && bx * TX + TX + 1 >= nx; --bx) ++hi;
  if (lo > tx) lo = tx;
}

// rank r of a tile CTA (dispatch order) -> natural tile index bx + tx (by + ty bz): the tx - lo - hi middle
// columns first, then the waiting columns
__device__ __forceinline__ int tile_of_rank(const TileGrid& G, int lo, int hi, int r) {
  const int mid = G.tx - lo - hi;
  const int nmid = mid * G.ty * G.tz;
  if (r < nmid) {
    const int rest = r / mid;
    return lo + (r - rest * mid) + G.tx * rest;
  }
  r -= nmid;
  const int w = lo + hi;
  const int rest = r / w, col = r - rest * w;
  return (col < lo ? col : G.tx - hi + (col - lo)) + G.tx * rest;
}

// The transfer CTAs occupy K1-sized slots (shared memory, registers) while they wait on memory, so there are few of
// them (at most XF_CTAS) and each thread loops over destination nodes, XF_U nodes per round: the map of the round's
// nodes (out, idx, xi) in one round of loads, then their 24 XF_U source loads at once.
constexpr int XF_CTAS = 48, XF_U = 2;
__host__ __device__ __forceinline__ int xfer_ctas(const FomLaunch& L) {
  long long n = 0;
  for (int m = 0; m < L.n_xf; ++m) n += L.xf[m].n;
  const long long c = (n + NT * XF_U - 1) / (NT * XF_U);
  return (int)(c < XF_CTAS ? c : XF_CTAS);
}

// K2 of the maps into this subdomain, s[p, c] = sum_{b<8} w_pb src[c cs + idx_pb] into X at out[3p + c] (P:L475-487,
// reading R11; the same arithmetic and order as transfer_kernel).  The sources' values it reads are fixed within the
// controller step (no donor corner on a source Schwarz DOF, or a ROM lift formed once per step, R39), so it runs
// beside the source's own K1.  Then the CTA signals xsync[0] (release).
__device__ __noinline__ void xfer_body(const FomLaunch& L, int blk, int tid) {
  const int n0 = L.xf[0].n;
  const int ntot = n0 + (L.n_xf > 1 ? L.xf[1].n : 0);
  const int stride = L.n_xf_ctas * NT;
  double* dst = const_cast<double*>(L.x);
  for (int t0 = blk * NT + tid; t0 < ntot; t0 += XF_U * stride) {
    int o[XF_U][3], id[XF_U][8];
    double xs[XF_U][3];
    const double* sb[XF_U];
    long long cs[XF_U];
#pragma unroll
    for (int u = 0; u < XF_U; ++u) {
      const int t = t0 + u * stride;
      const bool m0 = t < n0;
      const int p = m0 ? t : t - n0;
      o[u][0] = o[u][1] = o[u][2] = -1;
      sb[u] = m0 ? L.xf[0].src : L.xf[1].src;
      cs[u] = m0 ? L.xf[0].cs : L.xf[1].cs;
      if (t < ntot) {
        const int* out = (m0 ? L.xf[0].out : L.xf[1].out) + 3 * p;
        const int4* ix = reinterpret_cast<const int4*>((m0 ? L.xf[0].idx : L.xf[1].idx) + 8 * p);
        const double* xi = (m0 ? L.xf[0].xi : L.xf[1].xi) + 3 * p;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          o[u][c] = __ldg(out + c);
          xs[u][c] = __ldg(xi + c);
        }
        const int4 ia = __ldg(ix), ib = __ldg(ix + 1);
        id[u][0] = ia.x, id[u][1] = ia.y, id[u][2] = ia.z, id[u][3] = ia.w;
        id[u][4] = ib.x, id[u][5] = ib.y, id[u][6] = ib.z, id[u][7] = ib.w;
      }
    }
    double v[XF_U][3][8];
#pragma unroll
    for (int u = 0; u < XF_U; ++u)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < 8; ++q) v[u][c][q] = o[u][c] >= 0 ? __ldg(sb[u] + c * cs[u] + id[u][q]) : 0.0;
#pragma unroll
    for (int u = 0; u < XF_U; ++u)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double x = xs[u][0], y = xs[u][1], z = xs[u][2];
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double w = ((q & 1) ? x : 1.0 - x) * ((q & 2) ? y : 1.0 - y) * ((q & 4) ? z : 1.0 - z);
          a = fma(w, v[u][c][q], a);
        }
        if (o[u][c] >= 0) dst[o[u][c]] = a;
      }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(L.xsync) : "memory");
  }
}

// thread 0 of a waiting tile, before its first TMA issue: every transfer CTA of this launch is done (acquire; then
// the generic-proxy stores are ordered before the TMA reads).  The last of the n_wait waiters resets the handshake
// for the next launch.  A transfer CTA cannot be starved: CTAs are dispatched in index order and the transfer CTAs
// come first.  200 ms without them means a broken GPU: trap instead of hanging.
__device__ __noinline__ void xfer_wait(const FomLaunch& L, unsigned n_wait) {
  const unsigned long long t0 = global_ns();
  unsigned v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(L.xsync) : "memory");
    if (v >= (unsigned)L.n_xf_ctas) break;
    if (global_ns() - t0 > 200000000ULL) __trap();
    __nanosleep(128);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (atomicAdd(L.xsync + 1, 1u) == n_wait - 1) {
    L.xsync[0] = 0u;
    L.xsync[1] = 0u;
  }
}

// stage layout: X plane (halo box) | W plane (tile box) | W'_prev plane (tile box)
__device__ __forceinline__ void issue_plane(const TileGeo& P, bool wp, int it, int s, unsigned char* ring,
                                            unsigned long long* full, const Maps& M) {
  unsigned char* st = ring + (size_t)s * STAGE_BYTES;
  const int m = P.kbeg - 1 + it;
  mbar_expect_tx(&full[s], ARR_BYTES + (wp ? 2 : 1) * W_BYTES);
  tma_load_4d(st, M.x, P.x0, P.y0, m, 0, &full[s]);
  tma_load_4d(st + ARR_STRIDE, M.w, P.x0 + 2, P.y0 + 1, m, 0, &full[s]);
  if (wp) tma_load_4d(st + ARR_STRIDE + W_BYTES, M.wp, P.x0 + 2, P.y0 + 1, m, 0, &full[s]);
}

// One staged plane (iteration it of the tile, plane gi of the CTA's stream, staged plane
// m = kbeg - 1 + it).  Accumulator slots rotate by role: A = acc[SA] (node plane m+1), B = acc[SB]
// (plane m), C = acc[SC] (plane m-1, finished here if it lies in [kbeg, kend], then zeroed to become
// the next A).  Targets outside the chunk are accumulated too (and never used): every iteration is
// identical.
template <bool ZN, int SA, int SB, int SC>
__device__ __forceinline__ void k1_iter(const FomLaunch& L, const InteriorStencil& S, const Tile& T, int it, int gi,
                                        double (&acc)[3][3], double& num, double& den, unsigned char* ring,
                                        unsigned long long* full, unsigned long long* empty, const Maps& M) {
  const Geom& g = L.g;
  const int nz = g.nn[2] - 1;
  const long long np = g.npad;
  const int m = T.kbeg - 1 + it;
  const int kf = m - 1;
  const bool fin = T.writer() && kf >= T.kbeg && kf <= T.kend;
#ifdef OSAM_K1_PROF
  __shared__ long long k1prof[NWARP][4];
  const int kpw = ((int)threadIdx.x + TX * (int)threadIdx.y) >> 5;
  const bool kpl = (((int)threadIdx.x + TX * (int)threadIdx.y) & 31) == 0;
  if (it == 0 && kpl) k1prof[kpw][0] = k1prof[kpw][1] = k1prof[kpw][2] = k1prof[kpw][3] = 0;
  const long long kt0 = clock64();
#endif
  // producer (thread 0): plane it + NSTAGE - 2 into the stage released by plane it - 2.  One tile per CTA, so
  // the plane and its coordinates follow from the iteration and the thread's own tile constants (no cursor
  // in shared memory: c3 932 -> 953 steps/s; the role rotated over the warps, a non-blocking producer and an
  // issue at the end of the iteration were measured slower, profiles/r3_k1_experiments.md)
#if OSAM_K1_WARP
  // per-warp rings: lane 0 refills the stage its own warp released at the end of the previous iteration
  const bool issuer = (((int)threadIdx.x + TX * (int)threadIdx.y) & 31) == 0;
  if (issuer && it >= 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // its reads, then TMA
#else
  const bool issuer = threadIdx.x + threadIdx.y == 0;
#endif
  if (!PW && issuer && it + NSTAGE - 2 < T.nplanes) {
    const int p = it + NSTAGE - 2;
#if !defined(OSAM_K1_NOEMPTY) && !OSAM_K1_WARP  // NOEMPTY: probe only (wrong results)
    if (p >= NSTAGE) mbar_wait(&empty[p % NSTAGE], (unsigned)(((p - NSTAGE) / NSTAGE) & 1));
#endif
    TileGeo Pq;
    Pq.x0 = T.i - 2;
    Pq.y0 = T.j - 1;
    Pq.kbeg = T.kbeg;
    issue_plane(Pq, T.prev(), p, p % NSTAGE, ring, full, M);
  }
  const int s = gi % NSTAGE;
#ifdef OSAM_K1_PROF
  const long long kt1 = clock64();
#endif
  mbar_wait(&full[s], (unsigned)((gi / NSTAGE) & 1));
#ifdef OSAM_K1_PROF
  const long long kt2 = clock64();
#endif
  const double* xs = reinterpret_cast<const double*>(ring + (size_t)s * STAGE_BYTES);
  if (T.active()) {
    double* A = acc[SA];
    double* B = acc[SB];
    double* C = acc[SC];
    if (T.cy() == 1 && m >= 2 && m <= nz - 2) {
      plane_fast<true, true, true>(A, B, C, xs, pos_base(), S);
    } else {
      const Contrib3 r = plane_slow(xs, pos_base(), T.cy(), axis_class(m + 1, g.nn[2]), axis_class(m, g.nn[2]),
                                    axis_class(kf, g.nn[2]), L.rowc);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        A[c] += r.v[c];
        B[c] += r.v[3 + c];
        C[c] += r.v[6 + c];
      }
    }
  }
  if (T.active()) {
    const double* C = acc[SC];
    if (fin) {
      // own X, W, W'_prev of plane kf, staged in the previous iteration (released at the end of this one)
      const unsigned char* sp = ring + (size_t)((gi + NSTAGE - 1) % NSTAGE) * STAGE_BYTES;
      const double* xo = reinterpret_cast<const double*>(sp) + pos_own();
      const double* wo = reinterpret_cast<const double*>(sp + ARR_STRIDE) + pos_w();
      const double* qw = reinterpret_cast<const double*>(sp + ARR_STRIDE + W_BYTES) + pos_w();
      const long long id = T.id0 + (long long)kf * g.plane;
      const int cz = axis_class(kf, g.nn[2]);
      if (T.xface()) {  // fully constrained x-face node: Q' = X (prescribed), W' = a = 0
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (L.q_out) L.q_out[c * np + id] = xo[c * PLANE];
          L.w_out[c * np + id] = 0.0;
          if (L.a_out) L.a_out[c * np + id] = 0.0;
        }
      } else if (T.cy() == 1 && cz == 1 && L.a_out == nullptr && L.q_out != nullptr) {  // interior node
        const double inv_m = L.inv_mass[7];
        double* qo = L.q_out + id;
        double* wp = L.w_out + id;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double x = xo[c * PLANE], w0 = wo[c * WPL];
          const double an = -C[c] * inv_m;
          const double wn = fma(L.cw, an, w0);
          qo[c * np] = fma(L.cq, wn, x);
          wp[c * np] = wn;
          if (L.with_norm) {  // outside the band q = w' itself: d == 0 exactly (R38)
            const double w = fma(L.dt, fma(L.cv, an, w0), x);
            const double q = T.prev() ? qw[c * WPL] : (ZN ? w : wn);
            const double d = ZN ? w - q : 0.5 * L.dt * (wn - q);
            num = fma(d, d, num);
            den = fma(w, w, den);
          }
          if (ZN) L.z_out[c * np + id] = fma(L.dt, fma(L.cv, an, w0), x);
        }
      } else {
        const unsigned fm = (T.cy() != 1 || cz != 1) ? free_mask(g, L.f, T.i, T.j, kf) : 7u;
        const double inv_m = L.inv_mass[1 + 2 * (T.cy() == 1) + 4 * (cz == 1)];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double x = xo[c * PLANE];
          double an = 0.0, wn = 0.0, qn = x;
          if ((fm >> c) & 1) {
            const double w0 = wo[c * WPL];
            an = -C[c] * inv_m;
            wn = fma(L.cw, an, w0);
            qn = fma(L.cq, wn, x);
            if (L.with_norm) {
              const double w = fma(L.dt, fma(L.cv, an, w0), x);
              const double q = T.prev() ? qw[c * WPL] : (ZN ? w : wn);
              const double d = ZN ? w - q : 0.5 * L.dt * (wn - q);
              num = fma(d, d, num);
              den = fma(w, w, den);
            }
            if (ZN) L.z_out[c * np + id] = fma(L.dt, fma(L.cv, an, w0), x);
          }
          if (L.q_out) L.q_out[c * np + id] = qn;
          L.w_out[c * np + id] = wn;
          if (L.a_out) L.a_out[c * np + id] = an;
        }
      }
    }
  }
  // this warp is done with the previous plane of the stream (own values above, stencil before)
  __syncwarp();
  if (!OSAM_K1_WARP && gi >= 1 && (((int)threadIdx.x + TX * (int)threadIdx.y) & 31) == 0)
    mbar_arrive(&empty[(gi + NSTAGE - 1) % NSTAGE]);
#ifdef OSAM_K1_PROF
  if (kpl) {
    const long long kt3 = clock64();
    k1prof[kpw][0] += kt1 - kt0;
    k1prof[kpw][1] += kt2 - kt1;
    k1prof[kpw][2] += kt3 - kt2;
    if (it == T.nplanes - 1 && (blockIdx.x % 401) == 17)
      printf("K1PROF nx %d blk %d warp %d planes %d prod %lld wait %lld work %lld\n", L.g.nn[0], (int)blockIdx.x, kpw,
             T.nplanes, k1prof[kpw][0], k1prof[kpw][1], k1prof[kpw][2]);
  }
#endif
#pragma unroll
  for (int c = 0; c < 3; ++c) acc[SC][c] = 0.0;
}



__device__ __noinline__ void xface_body(const FomLaunch& L, int side_mask, int blk, int tid, int slot);

#ifndef OSAM_MINB
#define OSAM_MINB 4
#endif
#ifndef K1_MINB
#define K1_MINB OSAM_MINB
#endif

#ifndef OSAM_K1_ROT
// 0 (default): one copy of k1_iter per plane, the accumulator roles moved through the slots (9 moves per
// plane); 1: k1_iter unrolled by the period 3 of the roles (no moves).  The single copy keeps the loop in
// the instruction cache: c3 845 -> 891 steps/s (K1 0.203 -> 0.193 ms), 80 KB -> 54 KB of SASS, no spills.
#define OSAM_K1_ROT 0
#endif
template <bool ZN>
__global__ void __launch_bounds__(NTB, K1_MINB)
    fom_tiled_kernel(const __grid_constant__ FomLaunch L, const __grid_constant__ InteriorStencil S,
                     const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                     const __grid_constant__ CUtensorMap tmwp) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + NRING * NSTAGE * STAGE_BYTES);
  unsigned long long* empty = full + NRING * NSTAGE;
  if (L.stamp && threadIdx.x + threadIdx.y == 0) atomicMin(L.stamp, global_ns());  // in-schedule timeline
  const bool is_prod = PW && (int)threadIdx.y >= TY;  // the producer warp (whole warp: it may exit early)
  if (is_prod && ((int)blockIdx.x < L.n_xf_ctas || (int)blockIdx.x - L.n_xf_ctas >= L.n_tile_ctas)) return;
  if ((int)blockIdx.x < L.n_xf_ctas) {  // transfer CTAs (first)
    xfer_body(L, blockIdx.x, threadIdx.x + TX * threadIdx.y);
    if (L.stamp && threadIdx.x + threadIdx.y == 0) atomicMax(L.stamp + 1, global_ns());
    return;
  }
  const int b = (int)blockIdx.x - L.n_xf_ctas;  // = the partial slot of a tile (natural order) or x-face CTA
  if (b >= L.n_tile_ctas) {  // x-face CTAs (after the tile CTAs)
    xface_body(L, xface_sides(L.f), b - L.n_tile_ctas, threadIdx.x + TX * threadIdx.y, b);
    if (L.stamp && threadIdx.x + threadIdx.y == 0) atomicMax(L.stamp + 1, global_ns());
    return;
  }
  const Geom& g = L.g;
  const int nx = g.nn[0] - 1, ny = g.nn[1] - 1;
  const Maps M{&tmx, &tmw, &tmwp};
  const TileGrid G = tile_grid(g, L.f);
  // one CTA per tile; with the transfer in the grid the tiles that stage a Schwarz node come last and wait
  int t = b, wlo = 0, whi = 0;
  bool waits = false;
  if (L.n_xf_ctas) {
    wait_cols(g, L.f, G.tx, wlo, whi);
    t = tile_of_rank(G, wlo, whi, b);
    const int bx = t % G.tx;
    waits = bx < wlo || bx >= G.tx - whi;
  }
  const TileGeo P = tile_geo(g, G, t);
  Tile T;
  T.i = P.x0 + 2 + (int)threadIdx.x;
  T.j = P.y0 + 1 + (int)threadIdx.y;
  const bool active = (T.i <= nx) && (T.j <= ny);
  const bool xface = (T.i == 0) || (T.i == nx);
  const int xsd = T.i == 0 ? 0 : 1;
  const bool writer = active && (!xface || L.f.dir[xsd] == 7 || L.f.sw[xsd]);
  T.flags = (active ? 1u : 0u) | (xface ? 2u : 0u) | (writer ? 4u : 0u) | ((unsigned)axis_class(T.j, g.nn[1]) << 3) |
            (needs_prev(L, P) ? 32u : 0u);
  T.kbeg = P.kbeg;
  T.kend = P.kend;
  T.nplanes = P.nplanes;
  T.id0 = T.i + (long long)g.px * T.j;

#if OSAM_K1_WARP
  if (threadIdx.x + threadIdx.y == 0) {
    if (waits) xfer_wait(L, (unsigned)((wlo + whi) * G.ty * G.tz));
    for (int s = 0; s < NRING * NSTAGE; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  {
    const int w = ((int)threadIdx.x + TX * (int)threadIdx.y) >> 5;
    ring += (size_t)w * NSTAGE * STAGE_BYTES;
    full += w * NSTAGE;
    if ((((int)threadIdx.x + TX * (int)threadIdx.y) & 31) == 0) {
      TileGeo Pq = P;
      Pq.y0 = T.j - 1;  // the warp's first row - 1
      for (int p = 0; p < NSTAGE - 2 && p < T.nplanes; ++p) issue_plane(Pq, T.prev(), p, p, ring, full, M);
    }
  }
#else
  if (threadIdx.x + threadIdx.y == 0) {
    if (!PW && waits) xfer_wait(L, (unsigned)((wlo + whi) * G.ty * G.tz));
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    mbar_fence_init();
    if (!PW)
      for (int p = 0; p < NSTAGE - 2 && p < T.nplanes; ++p) issue_plane(P, T.prev(), p, p, ring, full, M);
  }
  __syncthreads();
  if (is_prod) {
    // the whole TMA stream of the tile: plane p goes into the stage plane p - NSTAGE left, released by the NWARP
    // consumer warps at the end of their iteration p - NSTAGE + 1 (the finish reads the previous stage)
    if (threadIdx.x == 0 && (int)threadIdx.y == TY) {
      if (waits) xfer_wait(L, (unsigned)((wlo + whi) * G.ty * G.tz));
      const bool wp = needs_prev(L, P);
#pragma unroll 1
      for (int p = 0; p < P.nplanes; ++p) {
        if (p >= NSTAGE) mbar_wait(&empty[p % NSTAGE], (unsigned)(((p - NSTAGE) / NSTAGE) & 1));
        issue_plane(P, wp, p, p % NSTAGE, ring, full, M);
      }
    }
    return;
  }
#endif

  double acc[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  double num = 0.0, den = 0.0;
#if OSAM_K1_ROT
  for (int it = 0; it < T.nplanes;) {  // unrolled by the period 3 of the slot rotation
    k1_iter<ZN, 0, 1, 2>(L, S, T, it, it, acc, num, den, ring, full, empty, M);
    if (++it >= T.nplanes) break;
    k1_iter<ZN, 2, 0, 1>(L, S, T, it, it, acc, num, den, ring, full, empty, M);
    if (++it >= T.nplanes) break;
    k1_iter<ZN, 1, 2, 0>(L, S, T, it, it, acc, num, den, ring, full, empty, M);
    ++it;
  }
#else
  // one copy of the iteration; the roles move through the slots (C, zeroed by k1_iter, becomes A)
#pragma unroll 1
  for (int it = 0; it < T.nplanes; ++it) {
    k1_iter<ZN, 0, 1, 2>(L, S, T, it, it, acc, num, den, ring, full, empty, M);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      acc[2][c] = acc[1][c];
      acc[1][c] = acc[0][c];
      acc[0][c] = 0.0;
    }
  }
#endif
  block_partial<NT>(num, den, L.partial, t);
  if (L.stamp && threadIdx.x + threadIdx.y == 0) atomicMax(L.stamp + 1, global_ns());
}

// Nodes on an x-face with free DOFs: a group of 4 lanes per node, lane sub = 0, 1, 2 gathers the
// plane oz = sub - 1 (6 positions: 2 in x, 3 in y; class-table stencil), the partial forces are summed
// in the order sub = 0, 1, 2 by shuffles and lane sub = 0 finishes the node.  side_mask bit 0: face
// x = 0, bit 1: face x = nx.
// Runs as the extra CTAs of the tiled kernel (blockIdx >= the tile CTAs), so it fills the tiled
// kernel's last wave instead of costing a launch of its own; blk = x-face block, slot = its partial slot.
__device__ __noinline__ void xface_body(const FomLaunch& L, int side_mask, int blk, int tid, int slot) {
  const Geom& g = L.g;
  const long long np = g.npad;
  const long long nf = (long long)g.nn[1] * g.nn[2];
  const int nsides = (side_mask & 1) + ((side_mask >> 1) & 1);
  const long long t = (blk * (long long)XF_BLOCK + tid) >> 2;
  const int sub = tid & 3;
  const int nx = g.nn[0] - 1;
  double num = 0.0, den = 0.0;
  const bool valid = t < nsides * nf;
  const int side = (side_mask == 2) ? 1 : (t >= nf ? 1 : 0);
  const long long r = t - (t >= nf ? nf : 0);
  const int i = side ? nx : 0;
  const int j = valid ? (int)(r % g.nn[1]) : 0;
  const int k = valid ? (int)(r / g.nn[1]) : 0;
  const int cyj = axis_class(j, g.nn[1]), czk = axis_class(k, g.nn[2]);
  double f[3] = {0.0, 0.0, 0.0};
  const int oz = sub - 1;
  if (valid && sub < 3 && k + oz >= 0 && k + oz <= g.nn[2] - 1) {
    const double* coef = L.coef + (size_t)((side ? 2 : 0) + 3 * (cyj + 3 * czk)) * 27 * 9;
    const int oxlo = side ? -1 : 0;
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy) {
      if (j + oy < 0 || j + oy > g.nn[1] - 1) continue;
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int ox = oxlo + dx;
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
  // fixed-order sum over the group: ((f_0 + f_1) + f_2)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double f1 = __shfl_down_sync(0xffffffffu, f[c], 1, 4);
    const double f2 = __shfl_down_sync(0xffffffffu, f[c], 2, 4);
    f[c] = (f[c] + f1) + f2;
  }
  if (valid && sub == 0) {
    const long long id = gidx(g, i, j, k);
    const unsigned fm = free_mask(g, L.f, i, j, k);
    const double inv_m = L.inv_mass[(cyj == 1 ? 2 : 0) + (czk == 1 ? 4 : 0)];
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
  block_partial<XF_BLOCK>(num, den, L.partial, slot);
}

long long tile_count(const Geom& g, const Faces& f) {
  return (long long)tile_cols(g, f) * cdiv(g.nn[1], TY) * cdiv(g.nn[2], ZC);
}

// CTAs of the tiled kernel: one per tile (a persistent variant, each resident CTA looping over tiles with one
// continuous TMA stream, measured equal in round 1 and was removed)
int tiled_ctas(const Geom& g, const Faces& f) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fom_tiled_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TILED);
    cudaFuncSetAttribute(fom_tiled_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TILED);
    attr = true;
  }
  return (int)tile_count(g, f);
}

unsigned xface_blocks(const Geom& g, const Faces& f) {
  const int m = xface_sides(f);
  const int ns = (m & 1) + ((m >> 1) & 1);
  return ns ? cdiv(4LL * ns * g.nn[1] * g.nn[2], XF_BLOCK) : 0u;
}

// the tiled kernel of one K1 (tile CTAs, then x-face CTAs)
void launch_tiled(const FomLaunch& L, const InteriorStencil& st, const CUtensorMap* tmx, const CUtensorMap* tmw,
                  const CUtensorMap* tmwp, cudaStream_t s) {
  FomLaunch Lt = L;
  Lt.n_tile_ctas = tiled_ctas(L.g, L.f);
  Lt.n_xf_ctas = L.n_xf > 0 ? xfer_ctas(L) : 0;
  // transfer CTAs, tile CTAs, then x-face CTAs
  const int grid = Lt.n_xf_ctas + Lt.n_tile_ctas + (int)xface_blocks(L.g, L.f);
  if (L.z_out)  // last substep of a multi-substep interval: z = u + dt v out, norm from z - z_prev (R33)
    fom_tiled_kernel<true><<<grid, dim3(TX, BY), SMEM_TILED, s>>>(Lt, st, *tmx, *tmw, *tmwp);
  else
    fom_tiled_kernel<false><<<grid, dim3(TX, BY), SMEM_TILED, s>>>(Lt, st, *tmx, *tmw, *tmwp);
  debug_check("fom_tiled_kernel", s);
}

int partial_slots(const Geom& g, const Faces& f) { return tiled_ctas(g, f) + (int)xface_blocks(g, f); }

// 4D (x, y, z, component) descriptor of a padded SoA field; halo = true: the X box (tile plus a
// 2/1-node halo in x/y), false: the W box (tile only).
int make_tmap(const Geom& g, double* array, bool halo, CUtensorMap* out) {
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
  const cuuint32_t box[4] = {halo ? (cuuint32_t)PX : (cuuint32_t)TX, halo ? (cuuint32_t)PY : (cuuint32_t)SR, 1, 3};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, array, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}
#undef K1_MINB
