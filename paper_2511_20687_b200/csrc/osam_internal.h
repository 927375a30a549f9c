// Internal types shared by the libosam.so translation units (host runtime + kernels).
// See include/osam.h for the public contract and DESIGN.md for the data layout.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <string>
#include <vector>

#include "../../include/osam.h"

namespace osam {

enum DofCode { DOF_FREE = 0, DOF_DIRICHLET = 1, DOF_SCHWARZ = 2 };

// Structured box geometry in the padded SoA layout used on the device:
//   field[c * npad + i + px * j + plane * k],  px = nn[0] rounded up to a multiple of 4
//   (component stride npad, z stride plane; see osam_create_subdomain for the two layouts).
struct Geom {
  int nn[3];
  int px;
  long long plane;  // z stride
  long long npad;   // component stride
  long long total;  // doubles per field
  double h[3];
  int small;        // the K1S gather path applies (OSAM_GATHER_MAX, decided at create and at bind)
};

// Per-subdomain boundary description passed to kernels by value.
struct Faces {
  unsigned char dir[6];  // Dirichlet component bitmask per face
  unsigned char sw[6];   // 1 if the face is a Schwarz face
  unsigned char shape;   // K1 tile shape 0: 32x4, 1: 16x8 (kernels_fom.cu k1_shape; decided at create and bind)
};

// 27 boundary classes x 27 neighbour offsets x 3x3 blocks of the merged hex8 stencil.
// class = cx + 3 (cy + 3 cz), c_d = 0 low face, 1 interior, 2 high face (per axis);
// offset = (ox+1) + 3((oy+1) + 3(oz+1)).
constexpr int NCLASS = 27;
// Interior-class stencil in parity-reduced form: k[slice][c][d] = {K(0,0), K(1,0), K(0,1), K(1,1)}
// at in-plane offsets (ox, oy), slice = oz + 1 (see kernels_fom.cu "parity-reduced stencil").
struct InteriorStencil {
  double k[3][3][3][4];
};

// Transfer map of one Schwarz face (destination) from one source.
struct XferMap {
  int src = -1;          // index of the source subdomain in the step group
  int face = -1;         // destination face
  int n = 0;             // destination nodes
  int* idx = nullptr;    // [n][8] source field indices (FOM: padded node id; ROM: compact lift id)
  double* xi = nullptr;  // [n][3] local coordinates in [0,1]
  int* out = nullptr;    // [n][3] destination index (FOM: c*npad + padded node id in q; ROM: Schwarz DOF
                         // id; -1 skip: Dirichlet component or a node owned by a lower Schwarz face)
  // multi-substep groups (R31): the source's trace over the controller interval,
  // [n_src_sub + 1 slots][B][3 n] (slot 0: the interval start), read through the interpolant Xi
  double* trace = nullptr;
  int n_src_sub = 1;
  // folded ROM-ROM exchange (groups of batched ROMs only, osam_api.cu bind_group): the destination's
  // reduced boundary input g^ = G u^_src with G = Phi_dS^T Pi Phi_src[donor rows] (r_b x r_src, column-
  // major), replacing lift, transfer and boundary projection
  double* G = nullptr;
  bool reads_src_schwarz = false;  // some donor corner is a Schwarz DOF of the source (its s enters)
};

struct Sub {
  // descriptor
  int kind = OSAM_FOM;
  double lo[3], hi[3];
  int nel[3];
  double E, nu, rho, lam, mu;
  unsigned char dirichlet[6];
  int batch = 1;
  int r = 0, r_b = 0;
  int n_sub = 1;      // substeps per controller step: dt_i = dt / n_sub
  int material = OSAM_LINEAR;  // FOM material (NL1 for SVK / Neohookean)
  double beta = 0.0;  // Newmark beta: 0 explicit, 1/4 implicit average acceleration (ROM only, R32)
  cudaStream_t stream = nullptr;
  Geom g;
  long long n_nodes = 0;

  // binding (first osam_step): Schwarz faces and DOF sets
  bool bound = false;
  std::vector<osam_subdomain*> group;
  int face_src[6] = {-1, -1, -1, -1, -1, -1};
  long long n_free = 0, n_sdof = 0;
  std::vector<int8_t> codes;  // host DOF codes (canonical DOF id 3p + c)
  std::vector<XferMap> maps;  // one per Schwarz face of this (destination) subdomain

  // FOM device state: buffers [3] x {q, w}, each 3 * npad doubles (R30).
  //   STEP state (w_dt > 0): st[cur] = (q, w) with q = u + w_dt w (boundary values in q) and
  //   w = v + w_dt/2 a; st[ux][0] = u of the checkpoint (exactly).
  //   RAW state (w_dt == 0, after osam_set_ic): st[cur] = (u, v).
  //   st[fr]: third buffer of the substep chain (allocated iff n_sub > 1).  Single-substep
  //   subdomains keep ux = 1 - cur.
  int cur = 0, ux = 1, fr = 2;
  double* st[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
  double* zbuf = nullptr;  // n_sub > 1: z = u + dt_i v of the last iterate's last substep (norm, R33)
  long long n_band = 0;    // nodes within one layer of a Schwarz face (the only ones whose norm term can
                           // change between iterations, R38)
  CUtensorMap tmapz;
  double w_dt = 0.0;
  Faces faces;
  double* coef = nullptr;  // device [NCLASS][27][9]
  double* rowc = nullptr;  // device row-form coefficients [cy][cz][slice][c][d][oy][2] (kernels_fom.cu)
  InteriorStencil stencil;
  CUtensorMap tmap[3];   // TMA descriptors of st[b][0] with the halo box (4D: x, y, z, component)
  CUtensorMap tmapw[3];  // TMA descriptors of st[b][1] with the tile box
  double mass_e = 0.0;  // rho * V_e / 8
  double inv_mass[8];   // 1 / (mass_e * prod_d (2 if interior on axis d else 1)), index cx + 2 cy + 4 cz
  double* scratch_v = nullptr;         // 3 * npad: v for osam_get_state
  double* scratch_a = nullptr;         // 3 * npad: acceleration for osam_get_accel
  double2* scratch_partial = nullptr;  // partial slots of non-sweep K1 launches
  unsigned* xsync = nullptr;           // [2] in-grid transfer handshake of the tiled K1 (FomLaunch::xsync)
  bool xin = false;                    // the transfers into it run as the first CTAs of its tiled K1 (bind)
  bool xpipe = false;                  // the transfers into it for sweep n + 1 follow its own advance of sweep n (bind)

  // ROM device data
  double *Phi = nullptr, *Phi_s = nullptr, *Kbar = nullptr, *Bbar = nullptr, *e = nullptr;
  std::vector<double> h_Phi, h_Phi_s, h_Kbar, h_Bbar, h_e;  // host copies (create)
  std::vector<double> h_Hbar, h_Cbar;  // polynomial OpInf terms (empty: absent)
  int order = 1;                       // 1 linear, 2 QOpInf, 3 COpInf
  int nf = 0;                          // polynomial features r(r+1)/2 [+ r(r+1)(r+2)/6]
  int* feat_idx = nullptr;             // device [nf][3] monomial indices (-1: unused third factor)
  double* F = nullptr;                 // device features [nf][B] (CUDA-core path)
  double* rst[2][4] = {{nullptr}};  // [buf] uh, vh, ah, s   (r x B, r x B, r x B, n_sdof x B)
  double* rsub[2][4] = {{nullptr}};  // n_sub > 1: intermediate substep states (same layout as rst)
  double* Minv = nullptr;            // implicit: [B][r][r] row-major (I + beta dt_i^2 e_b Kbar)^-1
  double* minv_work = nullptr;       // implicit: [B][r][2r] Gauss-Jordan scratch
  double minv_dt = 0.0;              // dt_i Minv was built for
  double* ustar = nullptr;          // r x B scratch
  double* gh = nullptr;             // r_b x B scratch
  int* free_ids = nullptr;          // n_free canonical DOF ids (device)
  int* sdof_ids = nullptr;          // n_sdof canonical DOF ids (device)
  // ROM as a transfer source: compact donor nodes and their lifted field [2][B][3][n_lift]
  std::vector<long long> lift_nodes;  // host, sorted node ids
  long long n_lift = 0;
  double* Phi_lift = nullptr;  // [3 n_lift][r] row-major
  int* lift_code = nullptr;    // [3 n_lift]: >= 0 Phi_lift row, -1 Dirichlet, -2-q Schwarz DOF q
  double* lift[2] = {nullptr, nullptr};
  std::vector<double> h_Phi_lift;  // host copy of Phi_lift (folding)
  bool fold = false;               // reduced boundary input from the folded operator of its map
  // batched ROM on the tensor cores (kernels_rom_tc.cu): [-Kbar | Bbar] and scratch
  bool use_tc = false;
  double* KB = nullptr;    // r x (r + r_b) column-major
  double* KBG = nullptr;   // folded exchange, linear explicit ROM: [-Kbar | Bbar G] (r x (r + r_src), column-major)
  // B = 1 ROM fed by one FOM map (c2): [-Kbar | Bbar G_F] row-major (r x (r + n_xd)), G_F = Phi_dS^T Pi restricted
  // to the n_xd source DOFs the map reads (xd_idx: their offsets in the source field); null: not folded
  double* KBF = nullptr;
  int* xd_idx = nullptr;
  int n_xd = 0;
  // explicit B = 1 ROM (CUDA-core path) whose exchange reads checkpoint-fixed data only (no map into it reads a
  // source Schwarz DOF, no map reading its lift reads its Schwarz DOFs): u~ and its lift are formed once per
  // controller step and its advance is a parallel graph branch (bind_group; implied by KBF)
  bool pre1 = false;
  double* KBr = nullptr;   // the same, row-major (CUDA-core path)
  double* Z = nullptr;     // (r + r_b) x B
  double* part = nullptr;  // split-K partial products (tc_part_size doubles)
  int* rp_cnt = nullptr;  // persistent batched-ROM controller: arrival counters of the update GEMM's C tiles

  // Phi given on a subset of its rows (osam.h phi_rows): the free-row index of each row of h_Phi,
  // ascending; empty = all n_free rows.  desc_n_free = the descriptor's n_free.
  std::vector<long long> h_phi_rows;
  long long desc_n_free = 0;

  // pending IC (raw full fields, batch x 3 n; or reduced: u^0, v^0 (r x B), s0 (n_s x B))
  bool ic_pending = false;
  bool ic_reduced = false;
  double* ic_u = nullptr;
  double* ic_v = nullptr;
  double* ic_s = nullptr;
};

// ---- kernel launchers (defined in the .cu files) ---------------------------------------
// One Schwarz transfer evaluated by the first CTAs of the destination's tiled K1 grid ("the
// transfer in the K1 grid"): s[p, c] = sum_b w_pb src[c cs + idx_pb] into the destination's X at out[3p + c].
struct XferPart {
  const int* idx;
  const double* xi;
  const int* out;
  const double* src;
  long long cs;
  int n;
};
constexpr int FOM_XF_MAX = 2;

struct FomLaunch {
  Geom g;
  Faces f;
  const double* x;   // staged field X (stencil input; TMA descriptor passed separately)
  const double* w0;  // per-node field W
  double* q_out;     // Q' = X + cq W' (may be null: not written)
  double* w_out;     // W' = W + cw a (also read first: previous iterate for the norm)
  double* z_out;     // optional: z = X + dt (W + cv a) out, and (with_norm) the norm from z - z_prev
                     // with z_prev staged from the same array (multi-substep intervals, R33)
  double* a_out;     // optional acceleration output (diagnostics), may be null
  double cw, cq;
  double cv;  // v = W + cv a (norm denominator)
  double dt;  // step in the convergence norm
  double inv_mass[8];
  const double* coef;  // [NCLASS][27][9]
  const double* rowc;  // [3][3][3][3][3][3][2] row-form coefficients
  int with_norm;       // 1 from Schwarz iteration 2 on
  double2* partial;    // per-block (num, den)
  int material;        // OSAM_LINEAR (K1) | OSAM_SVK | OSAM_NEOHOOKEAN (NL1)
  int n_tile_ctas;     // K1: CTAs that own tiles (set by launch_fom_advance; the rest do x-face work)
  unsigned long long* stamp;  // K1 in-schedule timeline (may be null): [0] earliest CTA start, [1] latest
                              // CTA end, %globaltimer ns (atomicMin / atomicMax); folded by K3, see Ctl
  double mat_lam, mat_mu, mat_kappa;
  // in-grid transfer (tiled K1 in a sweep, 0 otherwise): the first n_xf_ctas CTAs evaluate xf[0 .. n_xf) into x; the
  // tile CTAs whose staged box holds a Schwarz node run last and wait for them on xsync[0] (transfer CTAs done);
  // xsync[1] counts the waiters that passed, and the last one resets both
  XferPart xf[FOM_XF_MAX];
  int n_xf, n_xf_ctas;
  unsigned* xsync;
};
// Number of partial slots a K1 launch writes (tiled blocks + x-face blocks).
int fom_partial_slots(const Geom& g, const Faces& f);
// Can the transfers into this subdomain run as the first CTAs of its tiled K1 (Schwarz faces on x only, tiled
// linear path, and some tile column stages a Schwarz node)?
bool fom_ingrid_xfer_ok(const Geom& g, const Faces& f, int material);
int fom_nl_partial_slots(const Geom& g);  // NL1 (nonlinear materials): one slot per CTA
// with_xlast = false: the caller launches the excluded last x column (launch_fom_xlast) itself, e.g. on
// another stream concurrently with the tiled kernel (it reads only X and writes only that column).
void launch_fom_advance(const FomLaunch& L, const InteriorStencil& st, const CUtensorMap* tmx,
                        const CUtensorMap* tmw, const CUtensorMap* tmwp, cudaStream_t s, int* launches,
                        bool with_xlast = true);
void launch_fom_xlast(const FomLaunch& L, cudaStream_t s, int* launches);
// TMA descriptor of a padded SoA field for the K1 tile shape of (g, f) (halo: the X box, else the W box)
int make_field_tmap(const Geom& g, const Faces& f, double* array, bool halo, CUtensorMap* out);

void launch_transfer(const XferMap& m, const double* src, long long src_cstride, long long src_bstride,
                     double* dst, long long dst_bstride, int batch, const int* active, cudaStream_t s);
// multi-substep groups: Pi of the source field into trace slot `slot` of map m (compact [B][3n]),
// and the destination's Schwarz values at one of its substeps from the trace through Xi:
// (1 - alpha) trace[lo] + alpha trace[lo + 1]   (alpha == 0: trace[lo] as is)
void launch_transfer_trace(const XferMap& m, const double* src, long long src_cstride, long long src_bstride,
                           int slot, int batch, const int* active, cudaStream_t s);
void launch_trace_interp(const XferMap& m, int lo, double alpha, double* dst, long long dst_bstride, int batch,
                         const int* active, cudaStream_t s);
// implicit ROM: Minv[b] = (I + c e_b Kbar)^-1 by Gauss-Jordan with partial pivoting, one block per sample
void launch_rom_minv(int r, int B, const double* Kbar, const double* e, double c, double* work, double* Minv,
                     cudaStream_t s);
void launch_fom_pack(const Geom& g, const double* src_unpadded, double* dst_padded, long long n_nodes,
                     cudaStream_t s);
void launch_fom_unpack(const Geom& g, const double* src_padded, double* dst_unpadded, long long n_nodes,
                       cudaStream_t s);
void launch_fom_zero_constrained(const Geom& g, const Faces& f, double* u, double* w, cudaStream_t s);

struct RomLaunch {
  int r, r_b, B;
  long long n_sdof;
  const double *Phi_s, *Kbar, *Bbar, *e;
  const double* KBr;  // [-Kbar | Bbar | -Hbar | -Cbar] row-major r x (r + r_b + nf) (CUDA-core path)
  int nf;             // polynomial features (0: linear OpInf)
  const int* feat_idx;
  double* F;          // features [nf][B] (CUDA-core path)
  const double *uh0, *vh0, *ah0;  // checkpoint
  double *uh1, *vh1, *ah1;        // working
  const double* s;                // working Schwarz values (n_sdof x B)
  double *ustar, *gh;  // gh: partial g^ [gchunks][B][r_b] (CUDA-core path)
  int gchunks;
  const int* active;
  double dt;
  double c2;           // predictor u~ = u^ + dt v^ + c2 a^: dt^2/2 explicit, dt^2 (1/2 - beta) implicit
  double beta;         // 0: explicit; > 0: implicit average acceleration through Minv (R32)
  const double* Minv;  // [B][r][r] row-major
  const double* G;     // folded exchange: g^ = G Gu (r_b x Gr), null: g^ = Phi_dS^T s
  const double* Gu;    // the source's reduced state (Gr x B, column stride Gld; 0: Gr)
  int Gr;
  long long Gld;
  int pre;             // TC path: Z[0:r] (the predictor u~, and its features) was written at the step's start
  const double* KBG;   // TC path, pre: the update is [-Kbar | Bbar G] [u~; Gu] in one GEMM (null: G Gu first)
  int with_norm;
  double2* partial;
};
int rom_partial_slots(int r, bool tc);
int rom_gchunks(long long n_s);  // chunks of the partial boundary projection (CUDA-core path)
void launch_rom_advance(const RomLaunch& L, cudaStream_t s, int* launches);
void launch_rom_lift(int r, int B, long long n_lift, const double* Phi_lift, const int* code, const double* uh,
                     const double* s, long long n_sdof, double* out, cudaStream_t st);
cudaError_t launch_rom_project(long long n_rows, int r, int B, const double* Phi, const int* ids, const double* field,
                        long long field_bstride, long long n_nodes, double* out, cudaStream_t s);
void launch_gather_dofs(long long n, int B, const int* ids, const double* field, long long field_bstride,
                        long long n_nodes, double* out, cudaStream_t s);
void launch_rom_accel(const RomLaunch& L, const double* uh, double* ah, cudaStream_t s, int* launches);
// implicit polynomial ROM (R37): Newton per sample (rom_newton_kernel); shared memory it needs
size_t rom_newton_smem(int r, int r_b, int nf);
void launch_rom_newton(const RomLaunch& L, const double* ut, long long uts, const double* gsrc, long long gstride,
                       int gchunks, int n_slots, cudaStream_t s);
// implicit ROM finish (R32): a^' = Minv f (f in L.ah1), u^', v^', norm partials; u~ at ut (stride uts)
void launch_rom_implicit(const RomLaunch& L, const double* ut, long long uts, int n_slots, cudaStream_t s);
long long tc_part_size(int r, int r_b, int nf, int B, long long n_s, long long n_lift3);
long long tc_gemm_part(int M, int N, int K);  // split-K partial doubles of one M x N x K product
// F[q, b] = prod of u[idx[q][.], b]  (compressed Khatri-Rao monomials of the reduced state)
void launch_rom_features(int nf, int B, const int* idx, const double* u, long long ustride, double* F, long long fstride,
                         cudaStream_t s);
void launch_rom_advance_tc(const RomLaunch& L, const double* KB, double* Z, double* part, cudaStream_t s,
                           int* launches);
// Z[0:r] = u~ = u^ + dt v^ + c2 a^ of the checkpoint (and the polynomial features of u~), once per controller step
void launch_rom_predict_tc(const RomLaunch& L, double* Z, cudaStream_t s, int* launches);
// B = 1 ROM with the FOM exchange folded (KBF): a^' = e (-Kbar u~ + Bbar G_F x_d), x_d gathered from the source
// FOM field, u~ = L.ustar formed at the step's start; v^', u^', norm partials (one launch)
void launch_rom_fold_update(const RomLaunch& L, const double* KBF, const int* xd_idx, int n_xd, const double* src_field,
                            cudaStream_t s, int* launches);
void launch_rom_predict(const RomLaunch& L, cudaStream_t s, int* launches);  // L.ustar = u~ (CUDA-core path)
void launch_rom_accel_tc(const RomLaunch& L, const double* uh, double* ah, const double* KB, double* Z, double* part,
                         cudaStream_t s, int* launches);
void launch_rom_lift_tc(int r, int B, long long nl, const double* Phi_lift, const int* code, const double* uh,
                        const double* sv, long long ns, double* out, double* part, cudaStream_t st, int* launches);

// Batched subdomain-local OpInf replay (kernels_replay.cu, NEXT-4, reading R34).
struct ReplayArgs {
  int r, r_b, nf, B, K;
  double dt;
  const double* O;      // [B][r][r + r_b + nf] row-major
  const int* feat_idx;  // [nf][3]
  const double* Ubar;   // r x K column-major
  const double* Ghat;   // r_b x K column-major
  const double* vh0;    // r or null
  double* z;            // [B][r + r_b + nf] scratch
  double* traj;         // [B][K][r] or null
  double* err;          // [B]
  int* best;            // [1]
  int z_in_smem, o_in_smem;  // set by launch_replay
};
void launch_transpose_ops(int r, int rz, int B, const double* in_colmajor, double* out_rowmajor, cudaStream_t s);
cudaError_t launch_replay(ReplayArgs A, cudaStream_t s);


// Programmatic dependent launch (sm_90+): kernels launched with launch_k may be scheduled while their
// stream predecessor finishes; each such kernel calls pdl_enter() first (lets its own dependents launch,
// then waits for its predecessor's completion and memory), so the semantics are those of plain stream
// order and only the launch latency overlaps.  OSAM_PDL=0 disables the attribute.
inline bool pdl_enabled() {
  static const bool on = !(getenv("OSAM_PDL") && getenv("OSAM_PDL")[0] == '0');
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
#endif

// OSAM_DEBUG_SYNC=1: synchronise after every launch and report the first failing kernel on
// stderr (development aid only; off by default).
void debug_check(const char* kernel, cudaStream_t s);

struct Ctl {
  int* active;       // [B]
  int* iters;        // [B] of the current step
  double* numden;    // [B][2] last check
  int* flags;        // [0] any active, [1] unstable (this step)
  int* n_dev;        // Schwarz iterations done in the current step
  int* step_dev;     // controller steps started since the last reset
  int* sticky;       // [0] unstable, [1] hit max_iters (this osam_step call)
  int* iters_all;    // [steps][B] per-step iteration counts (may be null)
  double* trace;     // [steps][trace_T][B][2] (num, den) of every tested iteration n <= trace_T (may be null)
  int trace_T;
  // K1 timeline (may be null): stamps[2 i], [2 i + 1] = first start / last end of subdomain i's K1 in the
  // sweep that just ran; K3 adds, per sweep, busy[0] += the union of those intervals (ns), busy[1] += their
  // sum, busy[2] += launches, busy[3] += sweeps, busy[4] += sweeps n >= 2, and resets the stamps
  unsigned long long* stamps;
  int n_stamp;
  double* busy;
  int max_iters;
  int has_cond;      // graph mode: any_active sets the while-loop condition
  cudaGraphConditionalHandle cond;
};
void launch_step_begin(Ctl c, int B, cudaStream_t s);

// Persistent controller for small all-FOM groups (kernels_fom.cu small_persistent_kernel): one cooperative
// launch runs every controller step of an osam_step call -- the transfers in sweep order, the K1S node blocks
// of every subdomain, K3 and the controller flags, separated by grid-wide barriers -- with the buffer roles
// alternating by step parity on the device.
struct SmallMap {
  int n, src;
  const int *idx, *out;
  const double* xi;
};
struct SmallSub {
  FomLaunch L;           // template: geometry, faces, stencil table, masses, coefficients
  double* st[2][2];      // the two (q, w) buffers
  int slot0, nvb;        // first partial slot, K1S node blocks
  int cur0;              // checkpoint buffer index at the first step
  int n_maps;
  SmallMap maps[6];
};
constexpr int SMALL_MAX_SD = 4;
struct SmallArgs {
  int n_sd;
  SmallSub s[SMALL_MAX_SD];
  int n_steps;
  double tol_rel, tol_abs;
  int min_iters, max_iters;
  int n_slots;
  double2* partial;
  Ctl ctl;
  int* go;             // device int: the sweep loop continues (written by K3, read after the barrier)
  int res_coef_smem;   // small_resident_kernel: the class tables are staged in shared memory (set by its launcher)
};
cudaError_t launch_small_persistent(const SmallArgs& A, cudaStream_t s);
// The same group on one thread-block cluster with every subdomain's state in shared memory (kernels_fom.cu
// small_resident_kernel); cudaErrorNotSupported if it does not fit (OSAM_SMALL_RESIDENT=0: never).
cudaError_t launch_small_resident(const SmallArgs& A, cudaStream_t s);
int small_persistent_grid();  // CTAs that can be co-resident (cooperative launch bound)
bool fom_small(const Geom& g);  // the K1S (gather) path applies (g.small)
// Decide the FOM kernel path of a subdomain once (OSAM_GATHER_MAX -> g.small, OSAM_K1_SHAPE or the lane
// occupancy -> f.shape); called at create and at bind, before the TMA descriptors are encoded.
void choose_fom_path(Geom& g, Faces& f);

// Persistent controller for groups of batched tensor-core ROMs with the folded exchange (c5; kernels_rom_tc.cu
// rom_persistent_kernel): one cooperative launch runs every controller step of an osam_step call -- per ROM in
// sweep order (1) the predictor and the folded boundary input g^ = G u^_src, (2) the update GEMM [-Kbar | Bbar]
// [u~; g^] as split-K DMMA tiles whose last split runs the tile's epilogue (a^', v^', u^', norm partials), then K3
// and the controller flags for every sample -- two grid-wide barriers per ROM and one for K3 per sweep.
struct RomPSub {
  int r, rb, rz, Gr, src;
  const double *KB, *G, *e;
  double *Z, *part;
  int* cnt;                  // per C tile of the update GEMM: splits done (the last one runs the epilogue)
  double* rst[2][4];
  int slot0, cur0;
  int S_u, kc_u;             // split-K plan of the update GEMM (as gemm())
};
constexpr int ROMP_MAX_SD = 4;
struct RomPArgs {
  int n_sd, B;
  RomPSub s[ROMP_MAX_SD];
  int n_steps, min_iters, max_iters, n_slots;
  double dt, c2, tol_rel, tol_abs;
  double2* partial;
  Ctl ctl;
  int* go;
  unsigned* bar;  // [2] grid barrier (count, generation), zeroed before the launch
};
void rom_persist_plan(int r, int rb, int Gr, int B, RomPSub* p);  // split plan of the update GEMM (as gemm())
int rom_persist_slots(int r);           // norm partial slots of one ROM (one per 32-row tile)
int rom_persist_tiles(int r, int B);    // C tiles of the update GEMM (arrival counters)
cudaError_t launch_rom_persistent(const RomPArgs& A, cudaStream_t s);

// Convergence test of the sweep that just ran (iteration n = *n_dev + 1): K3 + flags/conditional.
// Returns the number of kernels launched (1 for a single sample: K3 and the flag update fused).
int launch_finalize(Ctl c, const double2* partial, int n_slots, int B, int min_iters, double tol_rel,
                    double tol_abs, cudaStream_t s);
// Groups of explicit batched tensor-core ROMs on the folded update (c5): the update GEMMs' epilogues (a^' from
// the split-K partials, v^', u^' = u~, the norm terms) and K3 in one launch, one block per sample; then the
// controller update.  Returns the launches.
struct EpiSub {
  const double* part;  // split-K partials of [-Kbar | Bbar G] [u~; u^_src]: part[z][i + r b]
  int S, r, rz;
  const double* Z;     // u~ in Z[0:r, b]
  const double *e, *ah0, *vh0;
  double *uh1, *vh1, *ah1;
};
struct EpiArgs {
  int n_sd, B;
  EpiSub s[4];
  double dt;
  int with_norm, min_iters;
  double tol_rel, tol_abs;
};
int launch_rom_epi_finalize(const EpiArgs& A, Ctl c, cudaStream_t s);
// the folded update GEMM alone (no epilogue); returns its number of K splits
int launch_rom_update_gemm_tc(const RomLaunch& L, double* Z, double* part, cudaStream_t s, int* launches);

}  // namespace osam
