// Host runtime of libosam.so: the C ABI of include/osam.h, subdomain binding (Schwarz-face
// detection and transfer maps), initial conditions, and the Schwarz controller that drives
// the kernels of kernels_fom.cu / kernels_xfer_rom.cu.
//
// Controller (Algorithm 1): for each controller step, sweep the subdomains in
// array order; a source that precedes the destination supplies iterate n, otherwise iterate
// n-1 (iterate 0 = its checkpoint: constant extension, reading R5); test convergence from
// n >= min_iters with eq:conv_criterion; commit by swapping the checkpoint and
// working buffers (no copy).  Hitting max_iters keeps the last iterate (reading R9).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <string>
#include <vector>

#include "osam_internal.h"

struct osam_subdomain {
  osam::Sub s;
};

namespace osam {
namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail(OSAM_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

template <class T>
int dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) return OSAM_OK;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? OSAM_ENOMEM : OSAM_ECUDA, "cudaMalloc(%zu bytes): %s",
                n * sizeof(T), cudaGetErrorString(e));
  }
  return OSAM_OK;
}
#define TRY(x)                 \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != OSAM_OK) return rc_; \
  } while (0)

template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// stream-ordered scratch (per-call buffers of offline routines: no device-wide synchronisation)
template <class T>
int dalloc_async(T** p, size_t n, cudaStream_t s) {
  *p = nullptr;
  const cudaError_t e = cudaMallocAsync((void**)p, std::max<size_t>(n, 1) * sizeof(T), s);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? OSAM_ENOMEM : OSAM_ECUDA, "cudaMallocAsync(%zu bytes): %s",
                n * sizeof(T), cudaGetErrorString(e));
  }
  return OSAM_OK;
}

template <class T>
void dfree_async(T*& p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
  p = nullptr;
}

}  // namespace

void debug_check(const char* kernel, cudaStream_t s) {
  static const bool on = getenv("OSAM_DEBUG_SYNC") != nullptr;
  if (!on) return;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "[osam debug] kernel %s failed: %s\n", kernel, cudaGetErrorString(e));
}

namespace {
// ---- profiling / launch accounting --------------------------------------------------------
bool g_prof = false;
double g_k1_ms = 0.0;
long long g_k1_launches = 0;
double g_k1_bytes = 0.0;
long long g_launches = 0;
int g_trace_T = 0;  // osam_set_conv_trace: record (num, den) of tested iterations n <= g_trace_T

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---- stencil coefficients (independent 1D tensor-product derivation) ---------------------
// Per axis and node class (0 low end, 1 interior, 2 high end) the assembled 1D rows of
//   M = int phi_p phi_q,  S = int phi_p' phi_q',  G = int phi_p' phi_q,  Gt = int phi_p phi_q'
// are the sums of the left- and right-element contributions that exist.  For a box mesh
// the 3D operator D_jl[p,q] = int d_j N_p d_l N_q factorises into per-axis rows (S on axis
// j = l; G on j and Gt on l for j != l; M elsewhere), and for isotropic elasticity
//   K_cd = lambda D_cd + mu delta_cd sum_l D_ll + mu D_dc      (A.1 P:L1939-1947).
void stencil_table(const double h[3], double lam, double mu, std::vector<double>& out) {
  double X[3][3][4][3];  // [axis][class][op M,S,G,Gt][offset+1]
  for (int ax = 0; ax < 3; ++ax) {
    const double hh = h[ax];
    const double L[4][3] = {{hh / 6, hh / 3, 0}, {-1 / hh, 1 / hh, 0}, {0.5, 0.5, 0}, {-0.5, 0.5, 0}};
    const double R[4][3] = {{0, hh / 3, hh / 6}, {0, 1 / hh, -1 / hh}, {0, -0.5, -0.5}, {0, -0.5, 0.5}};
    for (int cl = 0; cl < 3; ++cl) {
      const double eL = cl != 0 ? 1.0 : 0.0, eR = cl != 2 ? 1.0 : 0.0;
      for (int op = 0; op < 4; ++op)
        for (int o = 0; o < 3; ++o) X[ax][cl][op][o] = eL * L[op][o] + eR * R[op][o];
    }
  }
  out.assign((size_t)NCLASS * 27 * 9, 0.0);
  for (int cls = 0; cls < NCLASS; ++cls) {
    const int cl[3] = {cls % 3, (cls / 3) % 3, cls / 9};
    for (int off = 0; off < 27; ++off) {
      const int o[3] = {off % 3, (off / 3) % 3, off / 9};
      double D[3][3];
      for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l) {
          double v = 1.0;
          for (int ax = 0; ax < 3; ++ax) {
            const int op = (ax == j && ax == l) ? 1 : (ax == j ? 2 : (ax == l ? 3 : 0));
            v *= X[ax][cl[ax]][op][o[ax]];
          }
          D[j][l] = v;
        }
      const double tr = D[0][0] + D[1][1] + D[2][2];
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d)
          out[((size_t)cls * 27 + off) * 9 + c * 3 + d] = lam * D[c][d] + mu * (c == d ? tr : 0.0) + mu * D[d][c];
    }
  }
}

long long face_count(const Geom& g, int f) {
  const int ax = f >> 1;
  const int o0 = ax == 0 ? 1 : 0, o1 = ax == 2 ? 1 : 2;
  return (long long)g.nn[o0] * g.nn[o1];
}

// partial (num, den) slots of one FOM advance launch
int fom_slots(const Sub& s) {
  return s.material == OSAM_LINEAR ? fom_partial_slots(s.g, s.faces) : fom_nl_partial_slots(s.g);
}

// partial slots of a subdomain's advance: FOM blocks, ROM row groups (the folded FOM exchange: one per row)
int sub_slots(const Sub& s) {
  if (s.kind == OSAM_FOM) return fom_slots(s);
  return s.KBF ? s.r : rom_partial_slots(s.r, s.use_tc);
}

// ---- binding ------------------------------------------------------------------------------
void release_maps(Sub& s) {
  for (auto& m : s.maps) {
    dfree(m.idx);
    dfree(m.xi);
    dfree(m.out);
    dfree(m.trace);
    dfree(m.G);
  }
  s.maps.clear();
  s.fold = false;
}

void release_binding(Sub& s) {
  release_maps(s);
  dfree(s.scratch_partial);
  dfree(s.xsync);
  dfree(s.Phi);
  dfree(s.Phi_s);
  dfree(s.Kbar);
  dfree(s.Bbar);
  dfree(s.e);
  for (int b = 0; b < 2; ++b) {
    for (int q = 0; q < 4; ++q) {
      dfree(s.rst[b][q]);
      dfree(s.rsub[b][q]);
    }
    dfree(s.lift[b]);
  }
  dfree(s.Minv);
  dfree(s.minv_work);
  s.minv_dt = 0.0;
  dfree(s.ustar);
  dfree(s.gh);
  dfree(s.free_ids);
  dfree(s.sdof_ids);
  dfree(s.Phi_lift);
  dfree(s.lift_code);
  dfree(s.KB);
  dfree(s.KBG);
  dfree(s.KBF);
  dfree(s.xd_idx);
  s.n_xd = 0;
  dfree(s.KBr);
  dfree(s.feat_idx);
  dfree(s.F);
  dfree(s.Z);
  dfree(s.part);
  dfree(s.rp_cnt);
  s.bound = false;
  s.group.clear();
}

struct GraphKey {
  double dt, tol_rel, tol_abs;
  int max_iters, min_iters;
  std::vector<int> curs;
  bool operator<(const GraphKey& o) const {
    return std::tie(dt, tol_rel, tol_abs, max_iters, min_iters, curs) <
           std::tie(o.dt, o.tol_rel, o.tol_abs, o.max_iters, o.min_iters, o.curs);
  }
};

struct Group {
  std::vector<osam_subdomain*> sds;
  int B = 1;
  int n_slots = 0;
  double2* partial = nullptr;
  // device control block: [flags0, flags1, active[B], iters[B], n, step, sticky0, sticky1]
  int* ctl_i = nullptr;
  int* go = nullptr;  // persistent small-group controller: continue flag
  double* numden = nullptr;
  int* h_ctl = nullptr;  // pinned copy
  int* iters_all = nullptr;
  long long iters_cap = 0;
  unsigned long long* stamps = nullptr;  // K1 timeline stamps [n_sd][2] (Ctl::stamps)
  double* busy = nullptr;                // [5] K1 timeline accumulators (Ctl::busy)
  double2* ppartial = nullptr;           // norm partials of the persistent batched-ROM controller
  unsigned* rbar = nullptr;              // its grid barrier (count, generation)
  double* ctrace = nullptr;  // [steps][trace_T][B][2] convergence trace of the last osam_step call
  long long trace_cap = 0;
  int trace_T = 0, trace_steps = 0;
  std::vector<cudaEvent_t> ev;
  cudaStream_t cap_main = nullptr;    // private capture streams (the subdomains' stream may be the
  cudaStream_t cap_stream = nullptr;  // legacy default stream, which cannot be captured)
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int launches_per_sweep = 0;  // kernels of one sweep (launch accounting in graph mode)
  // FOM advances off the exchange's critical path (enqueue_sweep): one side stream and a fork / join
  // event pair per subdomain, in two sets (sweep 1 / the while-loop body: the body is captured while the
  // step graph's capture is still open, and a stream that joined one capture cannot join another)
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> fork_ev, join_ev;
  std::vector<cudaEvent_t> join2_ev, xl_ev;  // pipelined transfers: their end; the last-column copy's end
  int launches_begin = 1;      // kernels before sweep 1 (step_begin [+ trace slot 0])
  int unrolled = 0;            // sweeps 2 .. min_iters captured into the step graph itself (step_graph_capture)
  bool trace = false;          // some subdomain takes several substeps: transfers through traces + Xi
  int ctl_len() const { return 2 + 2 * B + 4; }
  ~Group() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (auto x : side) cudaStreamDestroy(x);
    for (auto e : fork_ev) cudaEventDestroy(e);
    for (auto e : join_ev) cudaEventDestroy(e);
    for (auto e : join2_ev) cudaEventDestroy(e);
    for (auto e : xl_ev) cudaEventDestroy(e);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (cap_main) cudaStreamDestroy(cap_main);
    dfree(partial);
    dfree(ctl_i);
    dfree(go);
    dfree(numden);
    dfree(iters_all);
    dfree(ctrace);
    dfree(stamps);
    dfree(busy);
    dfree(ppartial);
    dfree(rbar);
    if (h_ctl) cudaFreeHost(h_ctl);
    for (auto e : ev) cudaEventDestroy(e);
  }
  Ctl ctl(int max_iters) const {
    Ctl c;
    c.flags = ctl_i;
    c.active = ctl_i + 2;
    c.iters = ctl_i + 2 + B;
    c.n_dev = ctl_i + 2 + 2 * B;
    c.step_dev = ctl_i + 3 + 2 * B;
    c.sticky = ctl_i + 4 + 2 * B;
    c.numden = numden;
    c.iters_all = iters_all;
    c.trace = ctrace;
    c.trace_T = trace_T;
    c.stamps = stamps;
    c.n_stamp = (int)sds.size();
    c.busy = busy;
    c.max_iters = max_iters;
    c.has_cond = 0;
    c.cond = 0;
    return c;
  }
};
std::map<std::vector<osam_subdomain*>, std::unique_ptr<Group>> g_groups;

void forget_groups_with(osam_subdomain* h) {
  for (auto it = g_groups.begin(); it != g_groups.end();) {
    if (std::find(it->first.begin(), it->first.end(), h) != it->first.end())
      it = g_groups.erase(it);
    else
      ++it;
  }
}

// Schwarz faces: d_S Omega_i = d Omega_i cap Omega_j
void detect_faces(const std::vector<Sub*>& subs, int i, int face_src[6]) {
  const Sub& a = *subs[i];
  double size = 0;
  for (int d = 0; d < 3; ++d) size = std::max(size, a.hi[d] - a.lo[d]);
  const double tol = 1e-12 * size;
  for (int f = 0; f < 6; ++f) {
    face_src[f] = -1;
    const int ax = f / 2;
    const double x = (f & 1) ? a.hi[ax] : a.lo[ax];
    for (int j = 0; j < (int)subs.size(); ++j) {
      if (j == i) continue;
      const Sub& b = *subs[j];
      bool ok = b.lo[ax] + tol < x && x < b.hi[ax] - tol;
      for (int d = 0; d < 3 && ok; ++d)
        if (d != ax) ok = b.lo[d] <= a.lo[d] + tol && a.hi[d] <= b.hi[d] + tol;
      if (ok) {
        face_src[f] = j;
        break;
      }
    }
  }
}

void build_codes(Sub& s) {
  const Geom& g = s.g;
  s.codes.assign((size_t)3 * s.n_nodes, DOF_FREE);
  for (long long p = 0; p < s.n_nodes; ++p) {
    const int idx[3] = {(int)(p % g.nn[0]), (int)((p / g.nn[0]) % g.nn[1]), (int)(p / ((long long)g.nn[0] * g.nn[1]))};
    bool onf[6];
    for (int f = 0; f < 6; ++f) onf[f] = idx[f / 2] == ((f & 1) ? g.nn[f / 2] - 1 : 0);
    bool sw = false;
    for (int f = 0; f < 6; ++f) sw = sw || (onf[f] && s.face_src[f] >= 0);
    for (int c = 0; c < 3; ++c) {
      bool dir = false;
      for (int f = 0; f < 6; ++f) dir = dir || (onf[f] && ((s.dirichlet[f] >> c) & 1));
      s.codes[3 * p + c] = dir ? DOF_DIRICHLET : (sw ? DOF_SCHWARZ : DOF_FREE);
    }
  }
  s.n_free = s.n_sdof = 0;
  for (auto c : s.codes) {
    s.n_free += c == DOF_FREE;
    s.n_sdof += c == DOF_SCHWARZ;
  }
}

// owner Schwarz face of a node (lowest face index), -1 if none
int owner_face(const Sub& s, long long p) {
  const Geom& g = s.g;
  const int idx[3] = {(int)(p % g.nn[0]), (int)((p / g.nn[0]) % g.nn[1]), (int)(p / ((long long)g.nn[0] * g.nn[1]))};
  for (int f = 0; f < 6; ++f)
    if (s.face_src[f] >= 0 && idx[f / 2] == ((f & 1) ? g.nn[f / 2] - 1 : 0)) return f;
  return -1;
}

template <class T>
int upload(T** d, const std::vector<T>& h, cudaStream_t st) {
  TRY(dalloc(d, h.size()));
  if (!h.empty()) CK(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return OSAM_OK;
}

int process_ic(Sub& s, int* launches);

// TMA descriptors of a FOM's state buffers.  Their boxes follow the K1 tile shape, which depends on the
// faces (kernels_fom.cu k1_shape): encoded at create and again at bind, once the Schwarz faces are known.
int encode_tmaps(Sub& s) {
  choose_fom_path(s.g, s.faces);  // K1S vs tiled, tile shape: fixed with the descriptors
  const int nbuf = s.n_sub > 1 ? 3 : 2;
  for (int b = 0; b < nbuf; ++b) {
    int r = make_field_tmap(s.g, s.faces, s.st[b][0], true, &s.tmap[b]);
    if (r == 0) r = make_field_tmap(s.g, s.faces, s.st[b][1], false, &s.tmapw[b]);
    if (r == 0 && b == 0 && s.zbuf) r = make_field_tmap(s.g, s.faces, s.zbuf, false, &s.tmapz);
    if (r != 0) return r;
  }
  return 0;
}

int bind_group(const std::vector<Sub*>& subs, const std::vector<osam_subdomain*>& handles) {
  const int n = (int)subs.size();
  for (int i = 0; i < n; ++i) {
    release_binding(*subs[i]);
    detect_faces(subs, i, subs[i]->face_src);
    build_codes(*subs[i]);
  }
  // ROM shape checks and uploads
  for (int i = 0; i < n; ++i) {
    Sub& s = *subs[i];
    s.group = handles;
    if (s.kind != OSAM_ROM) {
      for (int f = 0; f < 6; ++f) {
        s.faces.dir[f] = s.dirichlet[f];
        s.faces.sw[f] = s.face_src[f] >= 0;
      }
      long long inner = 1;  // nodes farther than one layer from every Schwarz face
      for (int a = 0; a < 3; ++a)
        inner *= std::max(0, s.g.nn[a] - 2 * (int)s.faces.sw[2 * a] - 2 * (int)s.faces.sw[2 * a + 1]);
      s.n_band = s.n_nodes - inner;
      TRY(dalloc(&s.scratch_partial, (size_t)fom_slots(s)));
      TRY(dalloc(&s.xsync, 2));
      CK(cudaMemset(s.xsync, 0, 2 * sizeof(unsigned)));
      if (const int r = encode_tmaps(s)) return fail(OSAM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", r);
      continue;
    }
    const bool subset = !s.h_phi_rows.empty();
    const long long rows_phi = subset ? s.desc_n_free : (long long)(s.h_Phi.size() / std::max(1, s.r));
    const long long rows_phis = s.r_b > 0 ? (long long)(s.h_Phi_s.size() / s.r_b) : s.n_sdof;
    if (subset && s.h_phi_rows.back() >= s.n_free)
      return fail(OSAM_EINVAL, "ROM subdomain %d: phi_rows entry %lld >= n_free = %lld", i, s.h_phi_rows.back(),
                  s.n_free);
    if (rows_phi != s.n_free || rows_phis != s.n_sdof)
      return fail(OSAM_EINVAL, "ROM subdomain %d: Phi has %lld rows, Phi_s %lld, but the geometric split gives "
                  "n_free=%lld, n_s=%lld", i, rows_phi, rows_phis, s.n_free, s.n_sdof);
    if (s.r > s.n_free) return fail(OSAM_EINVAL, "ROM subdomain %d: r > n_free", i);
    std::vector<int> fid, sid;
    for (long long q = 0; q < 3 * s.n_nodes; ++q) {
      if (s.codes[q] == DOF_FREE) fid.push_back((int)q);
      if (s.codes[q] == DOF_SCHWARZ) sid.push_back((int)q);
    }
    if (!subset) TRY(upload(&s.Phi, s.h_Phi, s.stream));  // full Phi: the IC restriction u^0 = Phi^T u0
    TRY(upload(&s.Phi_s, s.h_Phi_s, s.stream));
    TRY(upload(&s.Kbar, s.h_Kbar, s.stream));
    TRY(upload(&s.Bbar, s.h_Bbar, s.stream));
    TRY(upload(&s.e, s.h_e, s.stream));
    TRY(upload(&s.free_ids, fid, s.stream));
    TRY(upload(&s.sdof_ids, sid, s.stream));
    for (int b = 0; b < 2; ++b) {
      for (int q = 0; q < 3; ++q) TRY(dalloc(&s.rst[b][q], (size_t)s.r * s.batch));
      TRY(dalloc(&s.rst[b][3], (size_t)std::max<long long>(1, s.n_sdof) * s.batch));
    }
    TRY(dalloc(&s.ustar, (size_t)s.r * s.batch));
    if (s.n_sub > 1)
      for (int b = 0; b < 2; ++b) {
        for (int q = 0; q < 3; ++q) TRY(dalloc(&s.rsub[b][q], (size_t)s.r * s.batch));
        TRY(dalloc(&s.rsub[b][3], (size_t)std::max<long long>(1, s.n_sdof) * s.batch));
      }
    if (s.beta > 0.0) {
      TRY(dalloc(&s.Minv, (size_t)s.r * s.r * s.batch));
      TRY(dalloc(&s.minv_work, (size_t)2 * s.r * s.r * s.batch));
    }
    TRY(dalloc(&s.gh, (size_t)std::max(1, s.r_b) * s.batch * rom_gchunks(s.n_sdof)));
    // batched samples: the reduced update is a dense contraction -> FP64 tensor cores (OSAM_ROM_TC=0/1
    // overrides the default, which is tensor cores iff batch > 1)
    const char* tc = getenv("OSAM_ROM_TC");
    s.use_tc = tc ? tc[0] == '1' : s.batch > 1;
    // reduced operator [-Kbar | Bbar | -Hbar | -Cbar] acting on z = [u^*; g^; u^*2; u^*3]
    // (eq:opinf_model_schwarz with the polynomial terms of eq:quadratic_opinf), column-major and
    // row-major copies, and the monomial index table of the compressed Khatri-Rao powers
    const int n2 = s.order >= 2 ? s.r * (s.r + 1) / 2 : 0;
    const int rz = s.r + s.r_b + s.nf;
    std::vector<double> kb((size_t)s.r * rz);
    for (int j = 0; j < s.r; ++j)
      for (int q = 0; q < s.r; ++q) kb[(size_t)j * s.r + q] = -s.h_Kbar[(size_t)j * s.r + q];
    for (int j = 0; j < s.r_b; ++j)
      for (int q = 0; q < s.r; ++q) kb[(size_t)(s.r + j) * s.r + q] = s.h_Bbar[(size_t)j * s.r + q];
    for (int j = 0; j < s.nf; ++j)
      for (int q = 0; q < s.r; ++q)
        kb[(size_t)(s.r + s.r_b + j) * s.r + q] =
            j < n2 ? -s.h_Hbar[(size_t)j * s.r + q] : -s.h_Cbar[(size_t)(j - n2) * s.r + q];
    std::vector<double> kbr((size_t)s.r * rz);
    for (int q = 0; q < s.r; ++q)
      for (int j = 0; j < rz; ++j) kbr[(size_t)q * rz + j] = kb[(size_t)j * s.r + q];
    TRY(upload(&s.KBr, kbr, s.stream));
    if (s.nf > 0) {
      std::vector<int> idx;
      for (int i = 0; i < s.r; ++i)
        for (int j = i; j < s.r; ++j) idx.insert(idx.end(), {i, j, -1});
      if (s.order >= 3)
        for (int i = 0; i < s.r; ++i)
          for (int j = i; j < s.r; ++j)
            for (int l = j; l < s.r; ++l) idx.insert(idx.end(), {i, j, l});
      TRY(upload(&s.feat_idx, idx, s.stream));
      TRY(dalloc(&s.F, (size_t)s.nf * s.batch));
    }
    if (s.use_tc) {
      TRY(upload(&s.KB, kb, s.stream));
      TRY(dalloc(&s.Z, (size_t)rz * s.batch));
    }
  }
  // donor maps: collect, per source, the nodes it must provide (ROM sources: compact lists)
  struct Pending {
    int dst, face, src;
    std::vector<long long> corner;  // [n][8] source node ids
    std::vector<double> xi;         // [n][3]
    std::vector<int> out;           // [n][3]
  };
  std::vector<Pending> pend;
  for (int i = 0; i < n; ++i) {
    Sub& d = *subs[i];
    for (int f = 0; f < 6; ++f) {
      const int j = d.face_src[f];
      if (j < 0) continue;
      const Sub& src = *subs[j];
      Pending P;
      P.dst = i;
      P.face = f;
      P.src = j;
      const int ax = f >> 1;
      const int o0 = ax == 0 ? 1 : 0, o1 = ax == 2 ? 1 : 2;
      const long long nf = face_count(d.g, f);
      P.corner.resize(nf * 8);
      P.xi.resize(nf * 3);
      P.out.resize(nf * 3);
      std::vector<long long> sdof_index;
      if (d.kind == OSAM_ROM) {
        sdof_index.assign((size_t)3 * d.n_nodes, -1);
        long long q = 0;
        for (long long t = 0; t < 3 * d.n_nodes; ++t)
          if (d.codes[t] == DOF_SCHWARZ) sdof_index[t] = q++;
      }
      for (long long t = 0; t < nf; ++t) {
        int idx[3];
        idx[ax] = (f & 1) ? d.g.nn[ax] - 1 : 0;
        idx[o0] = (int)(t % d.g.nn[o0]);
        idx[o1] = (int)(t / d.g.nn[o0]);
        const long long p = idx[0] + (long long)d.g.nn[0] * (idx[1] + (long long)d.g.nn[1] * idx[2]);
        int cell[3];
        for (int a = 0; a < 3; ++a) {
          const double X = d.lo[a] + idx[a] * d.g.h[a];
          const double tt = (X - src.lo[a]) / src.g.h[a];
          int ci = (int)std::floor(tt);
          ci = std::min(std::max(ci, 0), src.nel[a] - 1);
          const double x = tt - ci;
          if (!(x >= -1e-8 && x <= 1.0 + 1e-8))
            return fail(OSAM_EOVERLAP, "Schwarz node %lld of subdomain %d (face %d) lies outside source %d", p, i, f,
                        j);
          cell[a] = ci;
          P.xi[3 * t + a] = x;
        }
        for (int q = 0; q < 8; ++q) {
          const long long ci = cell[0] + (q & 1), cj = cell[1] + ((q >> 1) & 1), ck = cell[2] + ((q >> 2) & 1);
          P.corner[8 * t + q] = ci + (long long)src.g.nn[0] * (cj + (long long)src.g.nn[1] * ck);
        }
        for (int c = 0; c < 3; ++c) {
          // each Schwarz DOF is written by the map of its lowest Schwarz face; Dirichlet wins
          const bool mine = d.codes[3 * p + c] == DOF_SCHWARZ && owner_face(d, p) == f;
          if (!mine)
            P.out[3 * t + c] = -1;
          else if (d.kind == OSAM_ROM)
            P.out[3 * t + c] = (int)sdof_index[3 * p + c];
          else  // FOM: straight into the checkpoint's q (R30)
            P.out[3 * t + c] = (int)(c * d.g.npad + idx[0] + (long long)d.g.px * idx[1] + d.g.plane * idx[2]);
        }
      }
      pend.push_back(std::move(P));
    }
  }
  for (int j = 0; j < n; ++j) {
    Sub& s = *subs[j];
    if (s.kind != OSAM_ROM) continue;
    std::vector<long long> nodes;
    for (auto& P : pend)
      if (P.src == j) nodes.insert(nodes.end(), P.corner.begin(), P.corner.end());
    std::sort(nodes.begin(), nodes.end());
    nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
    s.lift_nodes = nodes;
    s.n_lift = (long long)nodes.size();
    const long long nl = 3 * s.n_lift;
    std::vector<long long> free_row((size_t)3 * s.n_nodes, -1), sidx((size_t)3 * s.n_nodes, -1);
    long long fr = 0, sr = 0;
    for (long long t = 0; t < 3 * s.n_nodes; ++t) {
      if (s.codes[t] == DOF_FREE) free_row[t] = fr++;
      if (s.codes[t] == DOF_SCHWARZ) sidx[t] = sr++;
    }
    std::vector<double> phil((size_t)std::max<long long>(nl, 1) * s.r, 0.0);
    std::vector<int> code((size_t)std::max<long long>(nl, 1), -1);
    for (int c = 0; c < 3; ++c)
      for (long long qi = 0; qi < s.n_lift; ++qi) {
        const long long ld = c * s.n_lift + qi;
        const long long dof = 3 * nodes[qi] + c;
        if (s.codes[dof] == DOF_FREE) {
          code[ld] = (int)ld;
          long long row = free_row[dof], ld_phi = s.n_free;  // row of h_Phi and its leading dimension
          if (!s.h_phi_rows.empty()) {  // Phi given on a subset of rows: the lift needs this one
            auto it = std::lower_bound(s.h_phi_rows.begin(), s.h_phi_rows.end(), row);
            if (it == s.h_phi_rows.end() || *it != row)
              return fail(OSAM_EINVAL, "ROM subdomain %d: the Schwarz transfer reads free row %lld of Phi, which is "
                          "not among phi_rows", j, row);
            row = (long long)(it - s.h_phi_rows.begin());
            ld_phi = (long long)s.h_phi_rows.size();
          }
          for (int k = 0; k < s.r; ++k) phil[ld * s.r + k] = s.h_Phi[row + (size_t)ld_phi * k];
        } else if (s.codes[dof] == DOF_SCHWARZ) {
          code[ld] = -2 - (int)sidx[dof];
        }
      }
    TRY(upload(&s.Phi_lift, phil, s.stream));
    s.h_Phi_lift = phil;
    TRY(upload(&s.lift_code, code, s.stream));
    for (int b = 0; b < 2; ++b) TRY(dalloc(&s.lift[b], (size_t)std::max<long long>(nl, 1) * s.batch));
    long long r_max = 0;  // a folded boundary GEMM contracts over the source's r instead of n_s
    for (int q = 0; q < n; ++q) r_max = std::max<long long>(r_max, subs[q]->r);
    if (s.use_tc)
      TRY(dalloc(&s.part, (size_t)tc_part_size(s.r, s.r_b, s.nf, s.batch, std::max(s.n_sdof, r_max), nl)));
  }
  // Folding ("algebraic folding is allowed"): in a group of batched tensor-core ROMs where
  // each ROM has one Schwarz map and no donor corner is a source Schwarz DOF (the lift would carry the
  // source's own s there), g^_dst = Phi_dS^T Pi (Phi_src[donor rows] u^_src) = G u^_src exactly up to
  // rounding: one small GEMM per sweep replaces the lift, the transfer and the boundary projection.
  bool fold = !getenv("OSAM_NO_FOLD") && n >= 2;
  for (int i = 0; i < n && fold; ++i) {
    const Sub& s = *subs[i];
    int maps_i = 0;
    for (auto& P : pend) maps_i += P.dst == i;
    fold = s.kind == OSAM_ROM && s.use_tc && s.n_sub == 1 && maps_i == 1 && s.r_b > 0;
  }
  for (auto& P : pend) {
    if (!fold) break;
    const Sub& src = *subs[P.src];
    for (size_t t = 0; t < P.out.size() && fold; ++t) {
      if (P.out[t] < 0) continue;
      const int c = (int)(t % 3);
      const long long p = (long long)(t / 3);
      for (int q = 0; q < 8; ++q)  // a donor corner on a source Schwarz DOF: the lift carries s there
        if (src.codes[3 * P.corner[8 * p + q] + c] == DOF_SCHWARZ) fold = false;
    }
  }
  for (auto& P : pend) {
    Sub& d = *subs[P.dst];
    const Sub& src = *subs[P.src];
    XferMap m;
    m.src = P.src;
    m.face = P.face;
    m.n = (int)(P.corner.size() / 8);
    std::vector<int> idx(P.corner.size());
    for (size_t q = 0; q < P.corner.size(); ++q) {
      const long long node = P.corner[q];
      if (src.kind == OSAM_ROM) {
        idx[q] = (int)(std::lower_bound(src.lift_nodes.begin(), src.lift_nodes.end(), node) - src.lift_nodes.begin());
      } else {
        const long long i0 = node % src.g.nn[0], j0 = (node / src.g.nn[0]) % src.g.nn[1],
                        k0 = node / ((long long)src.g.nn[0] * src.g.nn[1]);
        idx[q] = (int)(i0 + src.g.px * j0 + src.g.plane * k0);
      }
    }
    TRY(upload(&m.idx, idx, d.stream));
    TRY(upload(&m.xi, P.xi, d.stream));
    TRY(upload(&m.out, P.out, d.stream));
    m.n_src_sub = src.n_sub;
    for (size_t t = 0; t < P.out.size() && !m.reads_src_schwarz; ++t)
      if (P.out[t] >= 0)
        for (int q = 0; q < 8; ++q)
          if (src.codes[3 * P.corner[8 * (t / 3) + q] + (int)(t % 3)] == DOF_SCHWARZ) m.reads_src_schwarz = true;
    if (fold) {  // G[k + r_b j] = sum over the map's Schwarz DOFs and corners of Phi_dS[sd, k] w Phi_lift[row, j]
      const long long nl = src.n_lift;
      std::vector<double> G((size_t)d.r_b * src.r, 0.0);
      for (size_t t = 0; t < P.out.size(); ++t) {
        const int sd = P.out[t];
        if (sd < 0) continue;
        const int c = (int)(t % 3);
        const long long p = (long long)(t / 3);
        const double x = P.xi[3 * p], y = P.xi[3 * p + 1], z = P.xi[3 * p + 2];
        for (int q = 0; q < 8; ++q) {
          const double w = ((q & 1) ? x : 1.0 - x) * ((q & 2) ? y : 1.0 - y) * ((q & 4) ? z : 1.0 - z);
          const double* prow = src.h_Phi_lift.data() + (size_t)(c * nl + idx[8 * p + q]) * src.r;
          for (int k = 0; k < d.r_b; ++k) {
            const double a = d.h_Phi_s[(size_t)sd + (size_t)d.n_sdof * k] * w;
            if (a == 0.0) continue;
            double* gk = G.data() + k;
            for (int j = 0; j < src.r; ++j) gk[(size_t)d.r_b * j] += a * prow[j];
          }
        }
      }
      TRY(upload(&m.G, G, d.stream));
      d.fold = true;
      if (d.nf == 0 && d.beta == 0.0) {  // [-Kbar | Bbar G]: the whole reduced update of a linear explicit ROM
        const long long r = d.r, rs = src.r, rb = d.r_b;
        std::vector<double> kbg((size_t)(r * (r + rs)));
        for (long long j = 0; j < r; ++j)
          for (long long q = 0; q < r; ++q) kbg[(size_t)(j * r + q)] = -d.h_Kbar[(size_t)(j * r + q)];
        for (long long j = 0; j < rs; ++j)
          for (long long q = 0; q < r; ++q) {
            double a = 0.0;
            for (long long k = 0; k < rb; ++k) a += d.h_Bbar[(size_t)(k * r + q)] * G[(size_t)(k + rb * j)];
            kbg[(size_t)((r + j) * r + q)] = a;
          }
        TRY(upload(&d.KBG, kbg, d.stream));
        const long long need = tc_gemm_part(d.r, d.batch, d.r + src.r);
        long long rmx = 0;
        for (int q = 0; q < n; ++q) rmx = std::max<long long>(rmx, subs[q]->r);
        if (need > tc_part_size(d.r, d.r_b, d.nf, d.batch, std::max<long long>(d.n_sdof, rmx), 3 * d.n_lift)) {
          dfree(d.part);
          TRY(dalloc(&d.part, (size_t)need));
        }
      }
    }
    d.maps.push_back(m);
  }
  // B = 1 ROM fed by one FOM map that reads no source Schwarz DOF (c2): g^ = Phi_dS^T Pi x = G_F x_d exactly up
  // to rounding, x_d = the source DOFs the map reads; with the ROM's own update [-Kbar | Bbar G_F] acts on
  // [u~; x_d] (one small kernel per sweep instead of transfer + projection + update).  Needs the ROM's lift to
  // read no ROM Schwarz DOF (its s is then never formed) and an explicit single-substep linear ROM; groups with a
  // multi-substep subdomain keep the trace path.  OSAM_NO_FOLD disables it.
  bool any_sub = false, any_tc = false;
  for (int i = 0; i < n; ++i) {
    any_sub = any_sub || subs[i]->n_sub > 1;
    any_tc = any_tc || (subs[i]->kind == OSAM_ROM && subs[i]->use_tc);
  }
  for (int i = 0; i < n; ++i) {
    Sub& d = *subs[i];
    d.pre1 = false;
    if (any_sub || any_tc || getenv("OSAM_NO_PRE1") || d.kind != OSAM_ROM || d.batch != 1 || d.nf != 0 ||
        d.beta != 0.0)
      continue;
    bool ok = true;
    for (auto& mm : d.maps) ok = ok && !mm.reads_src_schwarz;
    for (int q = 0; q < n && ok; ++q)
      for (auto& mm : subs[q]->maps)
        if (mm.src == i && mm.reads_src_schwarz) ok = false;
    d.pre1 = ok;
  }
  // The transfers into a FOM run as the first CTAs of its tiled K1 ("the transfer in the K1 grid")
  // when every value they read is fixed within the controller step -- a FOM source's stencil input off its
  // Schwarz DOFs (R30), a pre1 ROM source's lift (R39) -- and no map reads this FOM's Schwarz DOFs (which the
  // in-grid transfer writes while other advances run).  Opt-in (OSAM_XFER_INGRID=1): measured slower than the
  // separate launches (c3 903 vs 970 steps/s), so the default keeps those.
  static const bool xin_env = getenv("OSAM_XFER_INGRID") && getenv("OSAM_XFER_INGRID")[0] == '1';
  for (int i = 0; i < n; ++i) {
    Sub& d = *subs[i];
    d.xin = false;
    if (!xin_env || any_sub || d.kind != OSAM_FOM || d.batch != 1 || d.maps.empty() ||
        (int)d.maps.size() > FOM_XF_MAX || !fom_ingrid_xfer_ok(d.g, d.faces, d.material))
      continue;
    bool ok = true;
    for (auto& mm : d.maps) {
      const Sub& src = *subs[mm.src];
      ok = ok && !mm.reads_src_schwarz && (src.kind == OSAM_FOM ? src.batch == 1 : src.pre1);
    }
    for (int q = 0; q < n && ok; ++q)
      for (auto& mm : subs[q]->maps)
        if (mm.src == i && mm.reads_src_schwarz) ok = false;
    d.xin = ok;
  }
  // Pipelined transfers: under the same conditions the transfers into a FOM for sweep n + 1 are
  // launched on its own branch right after its advance of sweep n (they write its Schwarz entries, which only that
  // advance reads), beside the other advances and K3 instead of ahead of the next sweep.  Every sweep still runs
  // every transfer; the one issued after the last sweep of a step rewrites the same bits (the values it reads are
  // fixed within the step from sweep 2 on).  OSAM_XFER_PIPE=0 keeps them at the head of their sweep.
  static const bool xpipe_env = !(getenv("OSAM_XFER_PIPE") && getenv("OSAM_XFER_PIPE")[0] == '0');
  for (int i = 0; i < n; ++i) {
    Sub& d = *subs[i];
    d.xpipe = false;
    if (!xpipe_env || d.xin || any_sub || d.kind != OSAM_FOM || d.batch != 1 || d.maps.empty()) continue;
    bool ok = true;
    for (auto& mm : d.maps) {
      const Sub& src = *subs[mm.src];
      ok = ok && !mm.reads_src_schwarz && (src.kind == OSAM_FOM ? src.batch == 1 : src.pre1);
    }
    for (int q = 0; q < n && ok; ++q)
      for (auto& mm : subs[q]->maps)
        if (mm.src == i && mm.reads_src_schwarz) ok = false;
    d.xpipe = ok;
  }
  // ... only in groups with one FOM (c2, c4: +1.4% on c4).  With two FOM advances in a sweep (c3) the second one's
  // transfers already run beside the first advance, and pipelining both (the two K1s start together: 965 vs 992
  // steps/s) or only the first (988 vs 996: the non-K1 time falls by 14 us per step but the K1s' union grows by
  // 22 us) measured slower (profiles/r7d_ab_xfer_pipe.log).  OSAM_XFER_PIPE=2 pipelines the first FOM of any group.
  static const bool xpipe_any = getenv("OSAM_XFER_PIPE") && getenv("OSAM_XFER_PIPE")[0] == '2';
  int n_fom = 0;
  for (int i = 0; i < n; ++i) n_fom += subs[i]->kind == OSAM_FOM;
  for (int i = 0, seen = 0; i < n; ++i)
    if (subs[i]->kind == OSAM_FOM) {
      if (seen++ || (n_fom > 1 && !xpipe_any)) subs[i]->xpipe = false;
    }
  for (auto& P : pend) {
    Sub& d = *subs[P.dst];
    const Sub& src = *subs[P.src];
    int maps_d = 0;
    for (auto& Q : pend) maps_d += Q.dst == P.dst;
    const bool ok = !getenv("OSAM_NO_FOLD") && d.pre1 && d.r_b > 0 && maps_d == 1 && src.kind == OSAM_FOM;
    if (!ok) continue;
    std::map<long long, int> col;  // source DOF offset -> column of x_d
    std::vector<int> xd;
    for (size_t t = 0; t < P.out.size(); ++t) {
      if (P.out[t] < 0) continue;
      const int c = (int)(t % 3);
      const long long p = (long long)(t / 3);
      for (int q = 0; q < 8; ++q) {
        const long long node = P.corner[8 * p + q];
        const long long i0 = node % src.g.nn[0], j0 = (node / src.g.nn[0]) % src.g.nn[1],
                        k0 = node / ((long long)src.g.nn[0] * src.g.nn[1]);
        const long long off = c * src.g.npad + i0 + src.g.px * j0 + src.g.plane * k0;
        if (col.emplace(off, (int)xd.size()).second) xd.push_back((int)off);
      }
    }
    const long long r = d.r, rb = d.r_b, nx = (long long)xd.size();
    if (r * (r + nx) > (4LL << 20)) continue;
    std::vector<double> G((size_t)(rb * nx), 0.0);  // G[k + rb t]
    for (size_t t = 0; t < P.out.size(); ++t) {
      const int sd = P.out[t];
      if (sd < 0) continue;
      const int c = (int)(t % 3);
      const long long p = (long long)(t / 3);
      const double x = P.xi[3 * p], y = P.xi[3 * p + 1], z = P.xi[3 * p + 2];
      for (int q = 0; q < 8; ++q) {
        const double w = ((q & 1) ? x : 1.0 - x) * ((q & 2) ? y : 1.0 - y) * ((q & 4) ? z : 1.0 - z);
        const long long node = P.corner[8 * p + q];
        const long long i0 = node % src.g.nn[0], j0 = (node / src.g.nn[0]) % src.g.nn[1],
                        k0 = node / ((long long)src.g.nn[0] * src.g.nn[1]);
        const int tc = col[c * src.g.npad + i0 + src.g.px * j0 + src.g.plane * k0];
        for (long long k = 0; k < rb; ++k) G[(size_t)(k + rb * tc)] += d.h_Phi_s[(size_t)sd + (size_t)d.n_sdof * k] * w;
      }
    }
    std::vector<double> kbf((size_t)(r * (r + nx)));  // row-major
    for (long long i = 0; i < r; ++i) {
      double* row = kbf.data() + (size_t)(i * (r + nx));
      for (long long j = 0; j < r; ++j) row[j] = -d.h_Kbar[(size_t)(j * r + i)];
      for (long long t = 0; t < nx; ++t) {
        double a = 0.0;
        for (long long k = 0; k < rb; ++k) a += d.h_Bbar[(size_t)(k * r + i)] * G[(size_t)(k + rb * t)];
        row[r + t] = a;
      }
    }
    TRY(upload(&d.KBF, kbf, d.stream));
    TRY(upload(&d.xd_idx, xd, d.stream));
    d.n_xd = (int)nx;
  }
  // multi-substep group: a trace of n_src_sub + 1 slots per map (R31)
  bool trace = false;
  int Bg = 1;
  for (int i = 0; i < n; ++i) {
    trace = trace || subs[i]->n_sub > 1;
    Bg = std::max(Bg, subs[i]->batch);
  }
  if (trace)
    for (int i = 0; i < n; ++i)
      for (auto& m : subs[i]->maps)
        TRY(dalloc(&m.trace, (size_t)(m.n_src_sub + 1) * Bg * 3 * std::max(1, m.n)));
  for (int i = 0; i < n; ++i) subs[i]->bound = true;
  int launches = 0;
  for (int i = 0; i < n; ++i)
    if (subs[i]->ic_pending) TRY(process_ic(*subs[i], &launches));
  g_launches += launches;
  return OSAM_OK;
}

// Initial condition once the Schwarz split is known (c.1 steps 8 and 10).
int process_ic(Sub& s, int* launches) {
  cudaStream_t st = s.stream;
  if (s.kind == OSAM_FOM) {
    // RAW state (u, v): Dirichlet u := 0, constrained v := 0; Schwarz DOFs keep u0.  a0 = -f(u0)/m
    // enters at the first osam_step (fom_set_step), once dt is known.
    launch_fom_zero_constrained(s.g, s.faces, s.st[s.cur][0], s.st[s.cur][1], st);
    *launches += 1;
    CK(cudaStreamSynchronize(st));
  } else {
    const int c = s.cur;
    if (s.ic_reduced) {  // osam_set_ic_reduced: u^0, v^0 (r x B) and s0 (n_s x B) as given
      if (s.ic_s == nullptr && s.n_sdof > 0)
        return fail(OSAM_EINVAL, "reduced IC: s0 missing although the subdomain has %lld Schwarz DOFs", s.n_sdof);
      CK(cudaMemcpyAsync(s.rst[c][0], s.ic_u, sizeof(double) * s.r * s.batch, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(s.rst[c][1], s.ic_v, sizeof(double) * s.r * s.batch, cudaMemcpyDeviceToDevice, st));
      if (s.n_sdof > 0)
        CK(cudaMemcpyAsync(s.rst[c][3], s.ic_s, sizeof(double) * s.n_sdof * s.batch, cudaMemcpyDeviceToDevice, st));
    } else {
      if (!s.Phi) return fail(OSAM_EINVAL, "ROM with a row subset of Phi: use osam_set_ic_reduced");
      const long long fbs = 3 * s.n_nodes;
      CK(launch_rom_project(s.n_free, s.r, s.batch, s.Phi, s.free_ids, s.ic_u, fbs, s.n_nodes, s.rst[c][0], st));
      CK(launch_rom_project(s.n_free, s.r, s.batch, s.Phi, s.free_ids, s.ic_v, fbs, s.n_nodes, s.rst[c][1], st));
      launch_gather_dofs(s.n_sdof, s.batch, s.sdof_ids, s.ic_u, fbs, s.n_nodes, s.rst[c][3], st);
    }
    RomLaunch L{};
    L.r = s.r;
    L.r_b = s.r_b;
    L.B = s.batch;
    L.n_sdof = s.n_sdof;
    L.Phi_s = s.Phi_s;
    L.Kbar = s.Kbar;
    L.Bbar = s.Bbar;
    L.KBr = s.KBr;
    L.nf = s.nf;
    L.feat_idx = s.feat_idx;
    L.F = s.F;
    L.e = s.e;
    L.s = s.rst[c][3];
    L.gh = s.gh;
    L.gchunks = rom_gchunks(s.n_sdof);
    if (s.use_tc) {
      launch_rom_accel_tc(L, s.rst[c][0], s.rst[c][2], s.KB, s.Z, s.part, st, launches);
      launch_rom_lift_tc(s.r, s.batch, 3 * s.n_lift, s.Phi_lift, s.lift_code, s.rst[c][0], s.rst[c][3], s.n_sdof,
                         s.lift[c], s.part, st, launches);
    } else {
      launch_rom_accel(L, s.rst[c][0], s.rst[c][2], st, launches);
      launch_rom_lift(s.r, s.batch, 3 * s.n_lift, s.Phi_lift, s.lift_code, s.rst[c][0], s.rst[c][3], s.n_sdof,
                      s.lift[c], st);
    }
    *launches += 4;
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaGetLastError());
  dfree(s.ic_u);
  dfree(s.ic_v);
  dfree(s.ic_s);
  s.ic_pending = false;
  s.ic_reduced = false;
  return OSAM_OK;
}

int get_group(osam_subdomain* const* sds, int n_sd, Group** out) {
  std::vector<osam_subdomain*> key(sds, sds + n_sd);
  auto it = g_groups.find(key);
  std::vector<Sub*> subs;
  for (auto h : key) subs.push_back(&h->s);
  bool need_bind = it == g_groups.end();
  for (auto s : subs) need_bind = need_bind || !s->bound || s->group != key;
  if (need_bind) {
    TRY(bind_group(subs, key));
    auto G = std::make_unique<Group>();
    G->sds = key;
    G->B = 1;
    for (auto s : subs) G->B = std::max(G->B, s->batch);
    for (auto s : subs) G->trace = G->trace || s->n_sub > 1;
    G->n_slots = 0;
    for (auto s : subs) G->n_slots += sub_slots(*s);
    TRY(dalloc(&G->partial, (size_t)std::max(1, G->n_slots) * G->B));
    TRY(dalloc(&G->ctl_i, (size_t)G->ctl_len()));
    CK(cudaMemset(G->ctl_i, 0, sizeof(int) * G->ctl_len()));
    TRY(dalloc(&G->numden, (size_t)2 * G->B));
    CK(cudaMallocHost((void**)&G->h_ctl, sizeof(int) * G->ctl_len()));
    {  // K1 timeline: stamps (start = ~0, end = 0) and zeroed accumulators
      std::vector<unsigned long long> st0(2 * G->sds.size());
      for (size_t q = 0; q < G->sds.size(); ++q) {
        st0[2 * q] = ~0ULL;
        st0[2 * q + 1] = 0ULL;
      }
      TRY(dalloc(&G->stamps, st0.size()));
      CK(cudaMemcpy(G->stamps, st0.data(), sizeof(unsigned long long) * st0.size(), cudaMemcpyHostToDevice));
      TRY(dalloc(&G->busy, 5));
      CK(cudaMemset(G->busy, 0, sizeof(double) * 5));
    }
    g_groups[key] = std::move(G);
    it = g_groups.find(key);
  }
  *out = it->second.get();
  return OSAM_OK;
}

// K1 launch description (kernels_fom.cu): stencil input X, per-node W, outputs Q', W' (, a).
FomLaunch fom_launch(const Sub& d, const double* x, const double* w0, double* q_out, double* w_out, double cw,
                     double cq, double cv, double dt, int with_norm, double2* partial, double* a_out) {
  FomLaunch L{};
  L.g = d.g;
  L.f = d.faces;
  L.x = x;
  L.w0 = w0;
  L.q_out = q_out;
  L.w_out = w_out;
  L.a_out = a_out;
  L.cw = cw;
  L.cq = cq;
  L.cv = cv;
  L.dt = dt;
  for (int q = 0; q < 8; ++q) L.inv_mass[q] = d.inv_mass[q];
  L.coef = d.coef;
  L.rowc = d.rowc;
  L.with_norm = with_norm;
  L.partial = partial;
  L.material = d.material;
  L.mat_lam = d.lam;
  L.mat_mu = d.mu;
  L.mat_kappa = d.lam + 2.0 * d.mu / 3.0;
  return L;
}

// Bring the state to STEP(dt) (R30), with a = -K u / m from one force pass:
//   RAW (u, v) in st[c]:    w = v + dt/2 a, q = u + dt w  -> st[ux]; st[c][0] keeps u; swap c, ux
//   STEP(dt0) in st[c]:     u = st[ux][0] exactly; w <- w + (dt - dt0)/2 a, q = u + dt w in place
// (dt: the subdomain step dt_i)
int fom_set_step(Sub& d, double dt, int* launches) {
  if (d.w_dt == dt) return OSAM_OK;
  const int c = d.cur, x = d.ux;
  if (d.w_dt == 0.0) {
    const FomLaunch L = fom_launch(d, d.st[c][0], d.st[c][1], d.st[x][0], d.st[x][1], 0.5 * dt, dt, 0.0,
                                   dt, 0, d.scratch_partial, nullptr);
    launch_fom_advance(L, d.stencil, &d.tmap[c], &d.tmapw[c], &d.tmapw[x], d.stream, launches);
    d.cur = x;
    d.ux = c;
  } else {
    const FomLaunch L = fom_launch(d, d.st[x][0], d.st[c][1], d.st[c][0], d.st[c][1], 0.5 * (dt - d.w_dt), dt,
                                   0.0, dt, 0, d.scratch_partial, nullptr);
    launch_fom_advance(L, d.stencil, &d.tmap[x], &d.tmapw[c], &d.tmapw[c], d.stream, launches);
  }
  d.w_dt = dt;
  return OSAM_OK;
}

// ROM advance description: state `in` -> `out` ({u^, v^, a^, s} buffers), step dt (= dt_i)
RomLaunch rom_launch(const Sub& d, double* const* in, double* const* out, const int* active, double dt,
                     int with_norm, double2* partial) {
  RomLaunch L{};
  L.r = d.r;
  L.r_b = d.r_b;
  L.B = d.batch;
  L.n_sdof = d.n_sdof;
  L.Phi_s = d.Phi_s;
  L.Kbar = d.Kbar;
  L.Bbar = d.Bbar;
  L.KBr = d.KBr;
  L.nf = d.nf;
  L.feat_idx = d.feat_idx;
  L.F = d.F;
  L.e = d.e;
  L.uh0 = in[0];
  L.vh0 = in[1];
  L.ah0 = in[2];
  L.uh1 = out[0];
  L.vh1 = out[1];
  L.ah1 = out[2];
  L.s = out[3];
  L.ustar = d.ustar;
  L.gh = d.gh;
  L.gchunks = rom_gchunks(d.n_sdof);
  L.active = active;
  L.dt = dt;
  L.c2 = d.beta > 0.0 ? (0.5 - d.beta) * dt * dt : 0.5 * dt * dt;
  L.beta = d.beta;
  L.Minv = d.Minv;
  L.with_norm = with_norm;
  L.partial = partial;
  return L;
}

// One Schwarz sweep of Algorithm 1 over the group, enqueued on `st`: for each
// subdomain in sweep order, K2 transfers from each source's current field (iterate n; at n = 1 a
// source later in the sweep supplies its checkpoint, reading R5), then the FOM advance K1 or the
// ROM advance K4-K6; finally K3 tests eq:conv_criterion and updates the device control
// block.  `first` selects the n = 1 variant (constant extension, no norm).
int enqueue_sweep_trace(Group& G, const osam_schwarz_cfg& cfg, const Ctl& ctl, bool first, cudaStream_t st,
                        int* launches, int* fom_k);

// side streams / events of the parallel FOM advances (created outside any stream capture)
int ensure_side(Group& G) {
  const int n = 2 * (int)G.sds.size();
  while ((int)G.side.size() < n) {
    cudaStream_t x;
    cudaEvent_t a, b, c, e;
    CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    G.side.push_back(x);
    G.fork_ev.push_back(a);
    G.join_ev.push_back(b);
    G.join2_ev.push_back(c);
    G.xl_ev.push_back(e);
  }
  return OSAM_OK;
}

int enqueue_sweep(Group& G, const osam_schwarz_cfg& cfg, const Ctl& ctl, bool first, cudaStream_t st, int* launches,
                  int* fom_k, bool main_set = false) {
  if (G.trace) return enqueue_sweep_trace(G, cfg, ctl, first, st, launches, fom_k);
  std::vector<Sub*> subs;
  for (auto h : G.sds) subs.push_back(&h->s);
  const int n_sd = (int)subs.size();
  const int B = G.B;
  int slot = 0;
  // In the explicit scheme a FOM iterate's displacement is its stencil input X (R30), so no transfer
  // reads a FOM advance's output: each FOM advance forks onto a side stream once its Schwarz values are
  // in and joins before the convergence test (parallel graph branches; their tails overlap).  Profiling
  // mode (per-launch K1 events) and OSAM_SERIAL_K1=1 keep them on the main stream.
  static const bool serial_env = getenv("OSAM_SERIAL_K1") && getenv("OSAM_SERIAL_K1")[0] == '1';
  const bool par = !g_prof && !serial_env;
  // side-stream set: 0 for sweeps captured into the step graph itself (sweep 1 and the unconditional sweeps up to
  // min_iters), n_sd for the while-loop body (captured while the step graph's capture is still open)
  const int set = (first || main_set) ? 0 : n_sd;
  if (par && (int)G.side.size() < 2 * n_sd) return fail(OSAM_ECUDA, "internal: side streams not created");
  std::vector<int> joins;
  // Groups of explicit batched tensor-core ROMs with the folded exchange (c5): an explicit ROM iterate's
  // displacement is its predictor u~ (u^' = u~), which depends on the checkpoint only, so u~ is formed once per
  // controller step (before sweep 1, into Z[0:r]) and a destination's folded input G u^_src reads the source's
  // Z[0:r] (its checkpoint u^ at n = 1 when the source comes later).  No ROM advance then reads another's output
  // within a sweep: each forks onto a side stream and joins before the test (parallel graph branches), as the FOM
  // advances do.  OSAM_ROM_PAR=0 keeps the serial chain.
  static const bool rom_par_env = !(getenv("OSAM_ROM_PAR") && getenv("OSAM_ROM_PAR")[0] == '0');
  bool rom_pre = rom_par_env && n_sd >= 2;
  for (int i = 0; i < n_sd && rom_pre; ++i) {
    const Sub& d = *subs[i];
    rom_pre = d.kind == OSAM_ROM && d.use_tc && d.fold && d.beta == 0.0 && d.n_sub == 1 && d.maps.size() == 1;
  }
  // B = 1 ROMs with the folded FOM exchange (KBF, c2): the explicit iterate's displacement is u~, formed once per
  // controller step with its lift (what the FOM's transfer reads from sweep 2 on); the ROM's update reads the
  // source FOM's field (its stencil input, fixed within the step at the DOFs the map reads) and no other
  // advance's output, so it runs as a parallel branch too
  // a pre1 ROM whose lift a later subdomain reads in sweep 1 (iterate 1 of an earlier source) forms u~ and the lift
  // here; the others do it on their own branch (the lift overlaps the FOM advance)
  auto lift_early = [&](int i) {
    for (int q = i + 1; q < n_sd; ++q)
      for (const XferMap& mm : subs[q]->maps)
        if (mm.src == i) return true;
    return false;
  };
  if (first)
    for (int i = 0; i < n_sd; ++i) {
      Sub& d = *subs[i];
      if (!d.pre1 || !lift_early(i)) continue;
      const RomLaunch L = rom_launch(d, d.rst[d.cur], d.rst[1 - d.cur], ctl.active, cfg.dt, 0, nullptr);
      launch_rom_predict(L, st, launches);
      launch_rom_lift(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, d.ustar, d.rst[1 - d.cur][3], d.n_sdof,
                      d.lift[1 - d.cur], st);
      *launches += d.n_lift > 0;
    }
  if (rom_pre && first)
    for (int i = 0; i < n_sd; ++i) {
      Sub& d = *subs[i];
      const RomLaunch L = rom_launch(d, d.rst[d.cur], d.rst[1 - d.cur], ctl.active, cfg.dt, 0, nullptr);
      launch_rom_predict_tc(L, d.Z, st, launches);
    }
  // ... and with every update folded ([-Kbar | Bbar G]), the epilogues run with K3 in one launch per sweep
  // (rom_epi_finalize_kernel; OSAM_EPI_FUSED=0: an epilogue per ROM, then K3)
  static const bool epi_env = !(getenv("OSAM_EPI_FUSED") && getenv("OSAM_EPI_FUSED")[0] == '0');
  static const bool kbg_env0 = !(getenv("OSAM_ROM_KBG") && getenv("OSAM_ROM_KBG")[0] == '0');
  bool epi_fused = rom_pre && kbg_env0 && epi_env && n_sd <= 4;
  for (int i = 0; i < n_sd && epi_fused; ++i) epi_fused = subs[i]->KBG != nullptr;
  EpiArgs epi{};
  for (int i = 0; i < n_sd; ++i) {
    Sub& d = *subs[i];
    // the transfers into d as the first CTAs of its K1 (bind: d.xin); in sweep 1 a later FOM source's iterate 0 is
    // its checkpoint u, the buffer its own K1 overwrites concurrently: separate launches before that K1 forks
    bool xin_now = d.xin;
    for (const XferMap& m : d.maps)
      if (first && m.src > i && subs[m.src]->kind == OSAM_FOM) xin_now = false;
    // pipelined transfers (bind: d.xpipe): from sweep 2 on the previous sweep issued them after this FOM's advance
    const bool xp = par && cfg.max_iters >= 2 && d.xpipe && !xin_now;
    for (const XferMap& m : d.maps) {
      if (d.fold || d.pre1 || xin_now || (xp && !first)) continue;  // folded: inside the ROM advance; pre1: below
      const Sub& src = *subs[m.src];
      const bool newest = (m.src < i) || !first;
      const double* field;
      long long cs, bs;
      if (src.kind == OSAM_FOM) {
        // a FOM iterate's displacement is its checkpoint q (predictor + current Schwarz values);
        // iterate 0 (constant extension) is the checkpoint u, kept in st[1-cur][0]
        field = newest ? src.st[src.cur][0] : src.st[src.ux][0];
        cs = src.g.npad;
        bs = 0;
      } else {
        field = src.lift[newest ? 1 - src.cur : src.cur];
        cs = src.n_lift;
        bs = 3 * src.n_lift;
      }
      double* dst;
      long long dbs;
      if (d.kind == OSAM_FOM) {
        dst = d.st[d.cur][0];
        dbs = 0;
      } else {
        dst = d.rst[1 - d.cur][3];
        dbs = d.n_sdof;
      }
      launch_transfer(m, field, cs, bs, dst, dbs, B, B > 1 ? ctl.active : nullptr, st);
      ++*launches;
    }
    const int with_norm = first ? 0 : 1;
    if (d.kind == OSAM_FOM) {
      const int c = d.cur, x = d.ux;
      FomLaunch L = fom_launch(d, d.st[c][0], d.st[c][1], d.st[x][0], d.st[x][1], cfg.dt, cfg.dt,
                               0.5 * cfg.dt, cfg.dt, with_norm, G.partial + (size_t)slot * B, nullptr);
      L.stamp = G.stamps + 2 * i;  // in-schedule K1 timeline (tiled K1; folded by K3)
      if (xin_now) {
        for (size_t q = 0; q < d.maps.size(); ++q) {
          const XferMap& m = d.maps[q];
          const Sub& src = *subs[m.src];
          const bool newest = (m.src < i) || !first;
          XferPart& xp = L.xf[q];
          xp.idx = m.idx;
          xp.xi = m.xi;
          xp.out = m.out;
          xp.n = m.n;
          if (src.kind == OSAM_FOM) {
            xp.src = newest ? src.st[src.cur][0] : src.st[src.ux][0];
            xp.cs = src.g.npad;
          } else {
            xp.src = src.lift[newest ? 1 - src.cur : src.cur];
            xp.cs = src.n_lift;
          }
        }
        L.n_xf = (int)d.maps.size();
        L.xsync = d.xsync;
      }
      cudaStream_t ks = st;
      if (par) {
        CK(cudaEventRecord(G.fork_ev[set + i], st));
        CK(cudaStreamWaitEvent(G.side[set + i], G.fork_ev[set + i], 0));
        ks = G.side[set + i];
        joins.push_back(set + i);
      }
      if (fom_k && g_prof) CK(cudaEventRecord(G.ev[2 * *fom_k], st));
      // the excluded last x column copies X there, Schwarz values included: after an in-grid transfer it follows K1
      launch_fom_advance(L, d.stencil, &d.tmap[c], &d.tmapw[c], &d.tmapw[x], ks, launches, !par || xin_now);
      if (fom_k && g_prof) CK(cudaEventRecord(G.ev[2 * *fom_k + 1], st));
      if (par) {
        CK(cudaEventRecord(G.join_ev[set + i], ks));
        if (!xin_now) launch_fom_xlast(L, st, launches);  // concurrently with the tiled kernel on the side stream
        if (xp) CK(cudaEventRecord(G.xl_ev[set + i], st));  // it reads X's last column, Schwarz values included
      }
      if (fom_k) ++*fom_k;
      // algorithmic bytes: read q, w and write q', w' (32 B/DOF) + the previous w' of the DOFs within one
      // layer of a Schwarz face from sweep 2 on (R38)
      g_k1_bytes += 32.0 * 3.0 * (double)d.n_nodes + (with_norm ? 8.0 * 3.0 * (double)d.n_band : 0.0);
      ++g_k1_launches;
      slot += fom_slots(d);
    } else {
      const int c = d.cur;
      RomLaunch L = rom_launch(d, d.rst[c], d.rst[1 - c], ctl.active, cfg.dt, with_norm,
                               G.partial + (size_t)slot * B);
      if (d.fold) {  // the source's iterate n if it precedes d, else n - 1 (n = 1: its checkpoint)
        const XferMap& m = d.maps[0];
        const Sub& src = *subs[m.src];
        const bool newest = (m.src < i) || !first;
        L.G = m.G;
        L.Gu = src.rst[newest ? 1 - src.cur : src.cur][0];
        L.Gr = src.r;
        if (rom_pre && newest) {  // = the source's predictor (explicit ROM), formed at the step's start
          L.Gu = src.Z;
          L.Gld = src.r + src.r_b + src.nf;
        }
      }
      if (d.KBF) {  // folded FOM exchange (B = 1): one kernel, a parallel branch
        const Sub& src = *subs[d.maps[0].src];
        cudaStream_t rs2 = st;
        if (par) {
          CK(cudaEventRecord(G.fork_ev[set + i], st));
          CK(cudaStreamWaitEvent(G.side[set + i], G.fork_ev[set + i], 0));
          rs2 = G.side[set + i];
          joins.push_back(set + i);
        }
        const bool late = first && !lift_early(i);
        if (late) launch_rom_predict(L, rs2, launches);
        launch_rom_fold_update(L, d.KBF, d.xd_idx, d.n_xd, src.st[src.cur][0], rs2, launches);
        if (late) {
          launch_rom_lift(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, d.ustar, d.rst[1 - d.cur][3], d.n_sdof,
                          d.lift[1 - d.cur], rs2);
          *launches += d.n_lift > 0;
        }
        if (par) CK(cudaEventRecord(G.join_ev[set + i], rs2));
        slot += sub_slots(d);
        continue;
      }
      if (d.pre1) {  // transfers into it, then its advance (the predictor formed at the step's start): a branch
        cudaStream_t rs2 = st;
        if (par) {
          CK(cudaEventRecord(G.fork_ev[set + i], st));
          CK(cudaStreamWaitEvent(G.side[set + i], G.fork_ev[set + i], 0));
          rs2 = G.side[set + i];
          joins.push_back(set + i);
        }
        for (const XferMap& m : d.maps) {
          const Sub& src = *subs[m.src];
          const bool newest = (m.src < i) || !first;
          const double* field;
          long long cs, bs;
          if (src.kind == OSAM_FOM) {
            field = newest ? src.st[src.cur][0] : src.st[src.ux][0];
            cs = src.g.npad;
            bs = 0;
          } else {
            field = src.lift[newest ? 1 - src.cur : src.cur];
            cs = src.n_lift;
            bs = 3 * src.n_lift;
          }
          launch_transfer(m, field, cs, bs, d.rst[1 - d.cur][3], d.n_sdof, B, nullptr, rs2);
          ++*launches;
        }
        L.pre = 1;
        const bool late = first && !lift_early(i);
        if (late) launch_rom_predict(L, rs2, launches);
        launch_rom_advance(L, rs2, launches);
        if (late) {
          launch_rom_lift(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, d.ustar, d.rst[1 - d.cur][3], d.n_sdof,
                          d.lift[1 - d.cur], rs2);
          *launches += d.n_lift > 0;
        }
        if (par) CK(cudaEventRecord(G.join_ev[set + i], rs2));
        slot += sub_slots(d);
        continue;
      }
      cudaStream_t rs = st;
      static const bool kbg_env = !(getenv("OSAM_ROM_KBG") && getenv("OSAM_ROM_KBG")[0] == '0');
      if (rom_pre && kbg_env) L.KBG = d.KBG;
      if (rom_pre && par) {
        L.pre = 1;
        CK(cudaEventRecord(G.fork_ev[set + i], st));
        CK(cudaStreamWaitEvent(G.side[set + i], G.fork_ev[set + i], 0));
        rs = G.side[set + i];
        joins.push_back(set + i);
      } else if (rom_pre) {
        L.pre = 1;
      }
      if (d.use_tc && epi_fused) {  // the update GEMM only; its epilogue runs with K3 below
        const int S = launch_rom_update_gemm_tc(L, d.Z, d.part, rs, launches);
        if (rs != st) CK(cudaEventRecord(G.join_ev[set + i], rs));
        EpiSub& es = epi.s[epi.n_sd++];
        es.part = d.part;
        es.S = S;
        es.r = d.r;
        es.rz = d.r + d.r_b + d.nf;
        es.Z = d.Z;
        es.e = d.e;
        es.ah0 = L.ah0;
        es.vh0 = L.vh0;
        es.uh1 = L.uh1;
        es.vh1 = L.vh1;
        es.ah1 = L.ah1;
      } else if (d.use_tc) {
        launch_rom_advance_tc(L, d.KB, d.Z, d.part, rs, launches);
        if (rs != st) CK(cudaEventRecord(G.join_ev[set + i], rs));
        if (!d.fold)  // in a folded group no map reads a lift
          launch_rom_lift_tc(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, d.rst[1 - c][0], d.rst[1 - c][3],
                             d.n_sdof, d.lift[1 - c], d.part, st, launches);
      } else {
        launch_rom_advance(L, st, launches);
        launch_rom_lift(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, d.rst[1 - c][0], d.rst[1 - c][3],
                        d.n_sdof, d.lift[1 - c], st);
        *launches += d.n_lift > 0;
      }
      slot += rom_partial_slots(d.r, d.use_tc);
    }
  }
  // pipelined transfers: the next sweep's Schwarz values of FOM i, on its branch after its advance (which alone
  // reads them); a ROM source's lift formed on that ROM's branch in sweep 1 is waited for
  std::vector<int> joins2;
  for (int i = 0; i < n_sd; ++i) {
    Sub& d = *subs[i];
    if (!(par && cfg.max_iters >= 2 && d.xpipe) || d.kind != OSAM_FOM) continue;
    cudaStream_t ks = G.side[set + i];
    CK(cudaStreamWaitEvent(ks, G.xl_ev[set + i], 0));
    for (const XferMap& m : d.maps) {
      const Sub& src = *subs[m.src];
      const double* field;
      long long cs, bs;
      if (src.kind == OSAM_FOM) {
        field = src.st[src.cur][0];
        cs = src.g.npad;
        bs = 0;
      } else {
        if (first && std::find(joins.begin(), joins.end(), set + m.src) != joins.end())
          CK(cudaStreamWaitEvent(ks, G.join_ev[set + m.src], 0));
        field = src.lift[1 - src.cur];
        cs = src.n_lift;
        bs = 3 * src.n_lift;
      }
      launch_transfer(m, field, cs, bs, d.st[d.cur][0], 0, B, nullptr, ks);
      ++*launches;
    }
    CK(cudaEventRecord(G.join2_ev[set + i], ks));
    joins2.push_back(set + i);
  }
  for (int i : joins) CK(cudaStreamWaitEvent(st, G.join_ev[i], 0));  // every FOM advance before the test
  if (epi_fused) {
    epi.B = B;
    epi.dt = cfg.dt;
    epi.with_norm = first ? 0 : 1;
    epi.min_iters = cfg.min_iters;
    epi.tol_rel = cfg.tol_rel;
    epi.tol_abs = cfg.tol_abs;
    *launches += launch_rom_epi_finalize(epi, ctl, st);
    return OSAM_OK;
  }
  *launches += launch_finalize(ctl, G.partial, G.n_slots, B, cfg.min_iters, cfg.tol_rel, cfg.tol_abs, st);
  for (int i : joins2) CK(cudaStreamWaitEvent(st, G.join2_ev[i], 0));  // the branches rejoin after K3
  return OSAM_OK;
}

// ---- multi-substep controller intervals (R31-R33) -----------------------------
// A subdomain with n_sub = m takes m steps of dt_i = dt/m per sweep.  FOM buffers: substep l reads
// X = (l == 0 ? st[cur] : output of substep l-1) and writes st[ux] (l even) / st[fr] (l odd); the
// last substep also writes z = u + dt_i v (norm, R33) when m > 1.  ROM: rst[cur] -> rsub[0/1] ->
// ... -> rst[1-cur].  Before substep l the Schwarz values at t + (l+1) dt_i are interpolated from
// each source's trace (Xi); after it, the subdomain's field at that time is projected into the
// trace slot l+1 of every map it feeds.

// Source field of a trace transfer: FOM -> the q array holding u (stride npad), ROM -> lift buffer.
void trace_source(const Sub& src, const double* field_fom, int lift_buf, const double** f, long long* cs,
                  long long* bs) {
  if (src.kind == OSAM_FOM) {
    *f = field_fom;
    *cs = src.g.npad;
    *bs = 0;
  } else {
    *f = src.lift[lift_buf];
    *cs = src.n_lift;
    *bs = 3 * src.n_lift;
  }
}

// Slot 0 of every trace: the sources' checkpoints (interval start).
int enqueue_trace_begin(Group& G, cudaStream_t st, int* launches) {
  std::vector<Sub*> subs;
  for (auto h : G.sds) subs.push_back(&h->s);
  for (auto sp : subs)
    for (const XferMap& m : sp->maps) {
      const Sub& src = *subs[m.src];
      const double* f;
      long long cs, bs;
      trace_source(src, src.kind == OSAM_FOM ? src.st[src.ux][0] : nullptr, src.cur, &f, &cs, &bs);
      launch_transfer_trace(m, f, cs, bs, 0, G.B, nullptr, st);
      ++*launches;
    }
  return OSAM_OK;
}

int enqueue_sweep_trace(Group& G, const osam_schwarz_cfg& cfg, const Ctl& ctl, bool first, cudaStream_t st,
                        int* launches, int* fom_k) {
  std::vector<Sub*> subs;
  for (auto h : G.sds) subs.push_back(&h->s);
  const int n_sd = (int)subs.size();
  const int B = G.B;
  const int* act = B > 1 ? ctl.active : nullptr;
  const int with_norm = first ? 0 : 1;
  int slot = 0;
  for (int i = 0; i < n_sd; ++i) {
    Sub& d = *subs[i];
    const int m = d.n_sub;
    const double dti = cfg.dt / m;
    double2* part = G.partial + (size_t)slot * B;
    for (int l = 0; l < m; ++l) {
      const bool last = l == m - 1;
      const int xb = l == 0 ? d.cur : ((l - 1) % 2 == 0 ? d.ux : d.fr);  // FOM input buffer
      const int ob = l % 2 == 0 ? d.ux : d.fr;                            // FOM output buffer
      double* const* rin = l == 0 ? d.rst[d.cur] : d.rsub[(l - 1) % 2];   // ROM states
      double* const* rout = last ? d.rst[1 - d.cur] : d.rsub[l % 2];
      // Schwarz values at t + (l+1) dt_i through Xi (R31); at n = 1 later sources give slot 0
      for (const XferMap& mp : d.maps) {
        int lo = 0;
        double alpha = 0.0;
        if (!(first && mp.src > i)) {
          const long long num = (long long)(l + 1) * mp.n_src_sub;
          lo = (int)(num / m);
          alpha = (double)(num % m) / (double)m;
        }
        if (d.kind == OSAM_FOM)
          launch_trace_interp(mp, lo, alpha, d.st[xb][0], 0, B, act, st);
        else
          launch_trace_interp(mp, lo, alpha, rout[3], d.n_sdof, B, act, st);
        ++*launches;
      }
      const double* field_fom = nullptr;
      if (d.kind == OSAM_FOM) {
        FomLaunch L = fom_launch(d, d.st[xb][0], d.st[xb][1], d.st[ob][0], d.st[ob][1], dti, dti, 0.5 * dti, dti,
                                 last ? with_norm : 0, part, nullptr);
        const bool zn = last && m > 1;
        if (zn) L.z_out = d.zbuf;
        if (fom_k && g_prof && last) CK(cudaEventRecord(G.ev[2 * *fom_k], st));
        launch_fom_advance(L, d.stencil, &d.tmap[xb], &d.tmapw[xb], zn ? &d.tmapz : &d.tmapw[ob], st, launches);
        if (fom_k && g_prof && last) {
          CK(cudaEventRecord(G.ev[2 * *fom_k + 1], st));
          ++*fom_k;
          g_k1_bytes += (32.0 + (L.with_norm ? 8.0 : 0.0) + (zn ? 8.0 : 0.0)) * 3.0 * (double)d.n_nodes;
          ++g_k1_launches;
        }
        field_fom = d.st[xb][0];  // u at t + (l+1) dt_i: the stencil input with its boundary values
      } else {
        const RomLaunch L = rom_launch(d, rin, rout, ctl.active, dti, last ? with_norm : 0, part);
        if (d.use_tc) {
          launch_rom_advance_tc(L, d.KB, d.Z, d.part, st, launches);
          launch_rom_lift_tc(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, rout[0], rout[3], d.n_sdof,
                             d.lift[1 - d.cur], d.part, st, launches);
        } else {
          launch_rom_advance(L, st, launches);
          launch_rom_lift(d.r, d.batch, 3 * d.n_lift, d.Phi_lift, d.lift_code, rout[0], rout[3], d.n_sdof,
                          d.lift[1 - d.cur], st);
          *launches += d.n_lift > 0;
        }
      }
      // this subdomain's field at t + (l+1) dt_i into slot l+1 of every map it feeds
      for (int e = 0; e < n_sd; ++e)
        for (const XferMap& mp : subs[e]->maps) {
          if (mp.src != i) continue;
          const double* f;
          long long cs, bs;
          trace_source(d, field_fom, 1 - d.cur, &f, &cs, &bs);
          launch_transfer_trace(mp, f, cs, bs, l + 1, B, act, st);
          ++*launches;
        }
    }
    slot += sub_slots(d);
  }
  *launches += launch_finalize(ctl, G.partial, G.n_slots, B, cfg.min_iters, cfg.tol_rel, cfg.tol_abs, st);
  return OSAM_OK;
}

// Commit a controller step: the working iterate becomes the checkpoint.  FOM buffer roles after m
// substeps (R30): m = 1: swap(cur, ux); m odd: (cur, ux, fr) <- (ux, fr, cur); m even: (fr, ux, cur).
void commit_step(Sub& d) {
  if (d.kind != OSAM_FOM) {
    d.cur = 1 - d.cur;
    return;
  }
  const int c = d.cur, x = d.ux, f = d.fr;
  if (d.n_sub == 1) {
    d.cur = x;
    d.ux = c;
  } else if (d.n_sub % 2 == 1) {
    d.cur = x;
    d.ux = f;
    d.fr = c;
  } else {
    d.cur = f;
    d.fr = c;
  }
}

// Host-driven controller step (profiling mode, or OSAM_NOGRAPH=1): the host reads the 16-byte
// convergence flags after every tested sweep.  Returns OSAM_OK / OSAM_WNOTCONVERGED / error.
int controller_step_host(Group& G, const osam_schwarz_cfg& cfg, cudaStream_t st) {
  int n_fom = 0;
  for (auto h : G.sds) n_fom += h->s.kind == OSAM_FOM;
  if (g_prof)
    while ((int)G.ev.size() < 2 * n_fom) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      G.ev.push_back(e);
    }
  const Ctl ctl = G.ctl(cfg.max_iters);
  int launches = 0;
  TRY(ensure_side(G));
  launch_step_begin(ctl, G.B, st);
  ++launches;
  if (G.trace) TRY(enqueue_trace_begin(G, st, &launches));
  bool done = false;
  for (int n = 1; n <= cfg.max_iters; ++n) {
    int fom_k = 0;
    TRY(enqueue_sweep(G, cfg, ctl, n == 1, st, &launches, &fom_k));
    if (n >= cfg.min_iters || g_prof) {
      CK(cudaMemcpyAsync(G.h_ctl, G.ctl_i, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (g_prof) {
        for (int k = 0; k < fom_k; ++k) {
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, G.ev[2 * k], G.ev[2 * k + 1]));
          g_k1_ms += ms;
        }
      }
      if (G.h_ctl[1]) {
        g_launches += launches;
        return fail(OSAM_EUNSTABLE, "non-finite Schwarz convergence norm at iteration %d", n);
      }
      if (n >= cfg.min_iters && !G.h_ctl[0]) {
        done = true;
        break;
      }
    }
  }
  CK(cudaGetLastError());
  for (auto h : G.sds) commit_step(h->s);  // commit: working iterate becomes the checkpoint
  g_launches += launches;
  return done ? OSAM_OK : OSAM_WNOTCONVERGED;
}

int step_graph_capture(Group& G, const osam_schwarz_cfg& cfg, cudaStream_t st, cudaGraph_t* graph_out,
                       int* launches_out) {
  Ctl ctl = G.ctl(cfg.max_iters);
  int launches = 0;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  cudaStreamCaptureStatus status;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t cap = nullptr;
  unsigned long long cap_id = 0;
  CK(cudaStreamGetCaptureInfo(st, &status, &cap_id, &cap, &deps, &ndeps));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, cap, cfg.max_iters >= 2 ? 1u : 0u, cudaGraphCondAssignDefault));
  launch_step_begin(ctl, G.B, st);
  int begin = 1;
  if (G.trace) TRY(enqueue_trace_begin(G, st, &begin));
  G.launches_begin = begin;
  TRY(enqueue_sweep(G, cfg, ctl, true, st, &launches, nullptr));
  // Sweeps 2 .. min_iters always run (the test starts at n = min_iters, R6/R7): they are captured into the step
  // graph itself, so a step pays the while-node's iteration overhead only from sweep min_iters + 1 on; their K3
  // sets the loop condition like the body's (no sample freezes and no error flag is raised before the first test at
  // n = min_iters, so the loop would have run them anyway).  Single-substep groups; OSAM_UNROLL_MIN=0 keeps every
  // sweep n >= 2 in the loop.
  static const bool unroll_env = !(getenv("OSAM_UNROLL_MIN") && getenv("OSAM_UNROLL_MIN")[0] == '0');
  G.unrolled = 0;
  if (unroll_env && !G.trace) {
    Ctl cu = ctl;
    cu.has_cond = 1;
    cu.cond = h;
    for (int n = 2; n <= cfg.min_iters && n <= cfg.max_iters; ++n) {
      int l2 = 0;
      TRY(enqueue_sweep(G, cfg, cu, false, st, &l2, nullptr, true));
      ++G.unrolled;
    }
  }
  CK(cudaStreamGetCaptureInfo(st, &status, &cap_id, &cap, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  CK(cudaGraphAddNode(&cnode, cap, deps, ndeps, &cp));
  CK(cudaStreamUpdateCaptureDependencies(st, &cnode, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(G.cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  ctl.has_cond = 1;
  ctl.cond = h;
  launches = 0;
  TRY(enqueue_sweep(G, cfg, ctl, false, G.cap_stream, &launches, nullptr));
  CK(cudaStreamEndCapture(G.cap_stream, &body));
  CK(cudaStreamEndCapture(st, graph_out));
  *launches_out = launches;
  return OSAM_OK;
}

// CUDA graph of one controller step: step_begin, sweep 1, then a conditional while node whose
// body is one sweep n >= 2; K3 (finalize_kernel) sets the loop condition on the device, so a step
// needs no host round trip.  One graph per (configuration, buffer parity), cached in the group.
int step_graph_capture(Group& G, const osam_schwarz_cfg& cfg, cudaStream_t st, cudaGraph_t* graph_out,
                       int* launches_out);

int step_graph(Group& G, const osam_schwarz_cfg& cfg, cudaStream_t, cudaGraphExec_t* out, int* launches_per_sweep) {
  GraphKey key{cfg.dt, cfg.tol_rel, cfg.tol_abs, cfg.max_iters, cfg.min_iters, {}};
  for (auto h : G.sds) {
    key.curs.push_back(h->s.cur);
    key.curs.push_back(h->s.ux);
  }
  auto it = G.graphs.find(key);
  if (it != G.graphs.end()) {
    *out = it->second;
    return OSAM_OK;
  }
  if (!G.cap_stream) CK(cudaStreamCreateWithFlags(&G.cap_stream, cudaStreamNonBlocking));
  if (!G.cap_main) CK(cudaStreamCreateWithFlags(&G.cap_main, cudaStreamNonBlocking));
  TRY(ensure_side(G));
  cudaGraph_t graph = nullptr;
  int launches = 0;
  const int rc = step_graph_capture(G, cfg, G.cap_main, &graph, &launches);
  if (rc != OSAM_OK) {  // leave no stream in capture mode
    cudaGraph_t junk = nullptr;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(G.cap_stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(G.cap_stream, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    junk = nullptr;
    if (cudaStreamIsCapturing(G.cap_main, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(G.cap_main, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
    return rc;
  }
  cudaGraphExec_t exec = nullptr;
  CK(cudaGraphInstantiate(&exec, graph, 0));
  CK(cudaGraphDestroy(graph));
  G.graphs[key] = exec;
  G.launches_per_sweep = launches;
  *out = exec;
  *launches_per_sweep = launches;
  return OSAM_OK;
}

int create_body(Sub& s, const osam_subdomain_desc* d, void* cuda_stream);
}  // namespace
}  // namespace osam

using namespace osam;

extern "C" {

const char* osam_last_error(void) { return g_err.c_str(); }

int osam_create_subdomain(const osam_subdomain_desc* d, void* cuda_stream, osam_subdomain** out) {
  if (!out) return fail(OSAM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!d) return fail(OSAM_EINVAL, "descriptor is NULL");
  if (d->kind != OSAM_FOM && d->kind != OSAM_ROM) return fail(OSAM_EINVAL, "kind must be OSAM_FOM or OSAM_ROM");
  for (int a = 0; a < 3; ++a) {
    if (!(d->hi[a] > d->lo[a])) return fail(OSAM_EINVAL, "hi <= lo on axis %d", a);
    if (d->nel[a] < 1) return fail(OSAM_EINVAL, "nel[%d] < 1", a);
  }
  if (!(d->E > 0) || !(d->rho > 0) || !(d->nu > -1.0 && d->nu < 0.5)) return fail(OSAM_EINVAL, "bad material");
  for (int f = 0; f < 6; ++f)
    if (d->dirichlet[f] > 7) return fail(OSAM_EINVAL, "dirichlet[%d] > 7", f);
  const long long nn0 = d->nel[0] + 1LL, nn1 = d->nel[1] + 1LL, nn2 = d->nel[2] + 1LL;
  if (nn0 * nn1 * nn2 > (1LL << 30)) return fail(OSAM_EINVAL, "mesh too large (> 2^30 nodes)");
  if (d->n_substeps < 0 || d->n_substeps > 4096) return fail(OSAM_EINVAL, "n_substeps must be in 0..4096");
  if (d->integrator != OSAM_EXPLICIT && d->integrator != OSAM_IMPLICIT)
    return fail(OSAM_EINVAL, "integrator must be OSAM_EXPLICIT or OSAM_IMPLICIT");
  if (d->kind == OSAM_FOM && d->integrator != OSAM_EXPLICIT)
    return fail(OSAM_EINVAL, "the FOM is explicit (implicit FOM solves are out of scope)");
  if (d->material != OSAM_LINEAR && d->material != OSAM_SVK && d->material != OSAM_NEOHOOKEAN)
    return fail(OSAM_EINVAL, "material must be OSAM_LINEAR, OSAM_SVK or OSAM_NEOHOOKEAN");
  if (d->kind == OSAM_ROM && d->material != OSAM_LINEAR)
    return fail(OSAM_EINVAL, "a ROM has no material model (its operators are inferred)");
  if (d->integrator == OSAM_IMPLICIT && (d->Hbar || d->Cbar)) {  // Newton in shared memory (R37)
    const long long r = d->r, n2 = r * (r + 1) / 2, n3 = d->Cbar ? r * (r + 1) * (r + 2) / 6 : 0;
    if (rom_newton_smem(d->r, d->r_b, (int)(n2 + n3)) > 200 * 1024)
      return fail(OSAM_EINVAL, "implicit polynomial ROM too large for the per-sample Newton solve (r = %d)", d->r);
  }
  if (d->kind == OSAM_ROM) {  // ROM descriptor checks (host-side, before any CUDA call)
    if (d->r < 1 || d->r_b < 0 || d->batch < 1) return fail(OSAM_EINVAL, "ROM needs r >= 1, r_b >= 0, batch >= 1");
    if (!d->Phi || !d->Kbar || (d->r_b > 0 && (!d->Phi_s || !d->Bbar)))
      return fail(OSAM_EINVAL, "ROM operator pointer is NULL");
    if (d->n_free < d->r || d->n_s < 0) return fail(OSAM_EINVAL, "ROM: n_free < r or n_s < 0");
    if (d->Cbar && !d->Hbar) return fail(OSAM_EINVAL, "Cbar (cubic OpInf) requires Hbar (quadratic term)");
  } else if (d->batch > 1) {
    return fail(OSAM_EINVAL, "a FOM subdomain has batch 1");
  }
  if (d->kind == OSAM_ROM && d->phi_rows) {  // Phi given on a subset of its rows (ascending free-row ids)
    if (d->n_phi_rows < d->r) return fail(OSAM_EINVAL, "ROM: n_phi_rows < r");
    for (int64_t q = 0; q < d->n_phi_rows; ++q)
      if (d->phi_rows[q] < 0 || d->phi_rows[q] >= d->n_free || (q > 0 && d->phi_rows[q] <= d->phi_rows[q - 1]))
        return fail(OSAM_EINVAL, "ROM: phi_rows must be strictly ascending in [0, n_free)");
  }
  {  // device offsets (transfer maps, TMA coordinates) are int32: 3 * padded nodes < 2^31
    const long long px = (nn0 + 3) / 4 * 4;
    if (3 * px * nn1 * nn2 >= (1LL << 31)) return fail(OSAM_EINVAL, "mesh too large (3 x padded nodes >= 2^31)");
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(OSAM_ECUDA, "cudaGetDevice: %s (no usable GPU)", cudaGetErrorString(e));

  auto h = std::make_unique<osam_subdomain>();
  const int rc = create_body(h->s, d, cuda_stream);
  if (rc != OSAM_OK) {  // frees whatever create_body allocated (no leak on any error path)
    osam_destroy(h.release());
    return rc;
  }
  *out = h.release();
  return OSAM_OK;
}

}  // extern "C"

namespace osam {
namespace {
int create_body(Sub& s, const osam_subdomain_desc* d, void* cuda_stream) {
  const long long nn0 = d->nel[0] + 1LL, nn1 = d->nel[1] + 1LL, nn2 = d->nel[2] + 1LL;
  s.kind = d->kind;
  for (int a = 0; a < 3; ++a) {
    s.lo[a] = d->lo[a];
    s.hi[a] = d->hi[a];
    s.nel[a] = d->nel[a];
  }
  s.E = d->E;
  s.nu = d->nu;
  s.rho = d->rho;
  s.lam = d->E * d->nu / ((1 + d->nu) * (1 - 2 * d->nu));
  s.mu = d->E / (2 * (1 + d->nu));
  std::memcpy(s.dirichlet, d->dirichlet, 6);
  s.stream = (cudaStream_t)cuda_stream;
  s.n_sub = std::max(1, (int)d->n_substeps);
  s.beta = d->integrator == OSAM_IMPLICIT ? 0.25 : 0.0;
  s.material = d->material;
  Geom& g = s.g;
  g.nn[0] = (int)nn0;
  g.nn[1] = (int)nn1;
  g.nn[2] = (int)nn2;
  g.px = (int)((nn0 + 3) / 4 * 4);
  // layout: the components interleaved per z-plane, [k][c][j][i]: component
  // stride npad (one component plane), z stride plane = 3 npad
  g.npad = (long long)g.px * nn1;
  g.plane = 3 * g.npad;
  g.total = g.plane * nn2;
  for (int a = 0; a < 3; ++a) g.h[a] = (d->hi[a] - d->lo[a]) / d->nel[a];
  s.n_nodes = nn0 * nn1 * nn2;
  s.mass_e = d->rho * g.h[0] * g.h[1] * g.h[2] / 8.0;
  for (int q = 0; q < 8; ++q)
    s.inv_mass[q] = 1.0 / (s.mass_e * ((q & 1) ? 2.0 : 1.0) * ((q & 2) ? 2.0 : 1.0) * ((q & 4) ? 2.0 : 1.0));
  std::memset(&s.faces, 0, sizeof s.faces);
  if (s.kind == OSAM_FOM) {
    s.batch = 1;
    std::vector<double> tab;
    stencil_table(g.h, s.lam, s.mu, tab);
    // parity-reduced interior stencil (kernels_fom.cu): K_cd(ox, oy, oz) = sx sy k[oz+1][c][d][|ox| + 2|oy|]
    // with sx = sign(ox) for blocks odd in x (exactly one of c, d is x), sy likewise in y, and the
    // oz = +1 slice equal to the oz = -1 slice times -1 for blocks odd in z.  Verified exactly.
    for (int sl = 0; sl < 3; ++sl)
      for (int c = 0; c < 3; ++c)
        for (int dd = 0; dd < 3; ++dd)
          for (int q = 0; q < 4; ++q) {
            const int off = (1 + (q & 1)) + 3 * ((1 + (q >> 1)) + 3 * sl);
            s.stencil.k[sl][c][dd][q] = tab[((size_t)13 * 27 + off) * 9 + c * 3 + dd];
          }
    for (int off = 0; off < 27; ++off) {
      const int o[3] = {off % 3 - 1, (off / 3) % 3 - 1, off / 9 - 1};
      for (int c = 0; c < 3; ++c)
        for (int dd = 0; dd < 3; ++dd) {
          const bool xodd = (c == 0) != (dd == 0), yodd = (c == 1) != (dd == 1), zodd = (c == 2) != (dd == 2);
          const int sl = o[2] == 1 ? 0 : o[2] + 1;
          double v = s.stencil.k[sl][c][dd][std::abs(o[0]) + 2 * std::abs(o[1])];
          if (xodd && o[0] == 0) v = 0.0;
          if (yodd && o[1] == 0) v = 0.0;
          if (xodd && o[0] < 0) v = -v;
          if (yodd && o[1] < 0) v = -v;
          if (zodd && o[2] == 0) v = 0.0;
          if (zodd && o[2] == 1) v = -v;
          if (v != tab[((size_t)13 * 27 + off) * 9 + c * 3 + dd])
            return fail(OSAM_EINVAL, "internal: interior stencil parity structure violated");
        }
    }
    // row form for face rows / face planes (kernels_fom.cu plane_slow), x-interior classes
    std::vector<double> rowc((size_t)27 * 54, 0.0);
    for (int cy = 0; cy < 3; ++cy)
      for (int cz = 0; cz < 3; ++cz)
        for (int sl = 0; sl < 3; ++sl) {
          const size_t cls = 1 + 3 * (cy + 3 * cz);
          for (int c = 0; c < 3; ++c)
            for (int dd = 0; dd < 3; ++dd)
              for (int oy = 0; oy < 3; ++oy) {
                auto K = [&](int ox) { return tab[(cls * 27 + (ox + 1) + 3 * (oy + 3 * sl)) * 9 + c * 3 + dd]; };
                const bool even = (c == 0) == (dd == 0);
                if (even ? K(-1) != K(1) : (K(-1) != -K(1) || K(0) != 0.0))
                  return fail(OSAM_EINVAL, "internal: face-class stencil x-parity violated");
                const size_t at = ((((size_t)(cy * 3 + cz) * 3 + sl) * 3 + c) * 3 + dd) * 3 + oy;
                rowc[2 * at] = even ? K(0) : 0.0;
                rowc[2 * at + 1] = K(1);
              }
        }
    TRY(upload(&s.rowc, rowc, s.stream));
    TRY(upload(&s.coef, tab, s.stream));
    TRY(dalloc(&s.scratch_a, (size_t)g.total));
    TRY(dalloc(&s.scratch_v, (size_t)g.total));
    const int nbuf = s.n_sub > 1 ? 3 : 2;  // substep chains need a third (q, w) buffer and z
    for (int b = 0; b < nbuf; ++b)
      for (int q = 0; q < 2; ++q) {
        TRY(dalloc(&s.st[b][q], (size_t)g.total));
        CK(cudaMemsetAsync(s.st[b][q], 0, sizeof(double) * g.total, s.stream));
      }
    if (s.n_sub > 1) {
      TRY(dalloc(&s.zbuf, (size_t)g.total));
      CK(cudaMemsetAsync(s.zbuf, 0, sizeof(double) * g.total, s.stream));
    }
    const int r = encode_tmaps(s);
    if (r != 0) return fail(OSAM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", r);
  } else {
    s.r = d->r;
    s.r_b = d->r_b;
    s.batch = d->batch;
    s.desc_n_free = d->n_free;
    if (d->phi_rows) {
      s.h_phi_rows.assign(d->phi_rows, d->phi_rows + d->n_phi_rows);
      s.h_Phi.assign(d->Phi, d->Phi + (size_t)d->n_phi_rows * d->r);
    } else {
      s.h_Phi.assign(d->Phi, d->Phi + (size_t)d->n_free * d->r);
    }
    if (d->r_b > 0) {
      s.h_Phi_s.assign(d->Phi_s, d->Phi_s + (size_t)d->n_s * d->r_b);
      s.h_Bbar.assign(d->Bbar, d->Bbar + (size_t)d->r * d->r_b);
    }
    s.h_Kbar.assign(d->Kbar, d->Kbar + (size_t)d->r * d->r);
    s.order = d->Cbar ? 3 : (d->Hbar ? 2 : 1);
    const long long n2 = (long long)d->r * (d->r + 1) / 2, n3 = (long long)d->r * (d->r + 1) * (d->r + 2) / 6;
    if (s.order >= 2) s.h_Hbar.assign(d->Hbar, d->Hbar + (size_t)d->r * n2);
    if (s.order >= 3) s.h_Cbar.assign(d->Cbar, d->Cbar + (size_t)d->r * n3);
    s.nf = (int)((s.order >= 2 ? n2 : 0) + (s.order >= 3 ? n3 : 0));
    s.h_e.assign((size_t)d->batch, 1.0);
    if (d->e_scale)
      for (int b = 0; b < d->batch; ++b) s.h_e[b] = d->e_scale[b];
    if (d->r_b == 0) s.h_Phi_s.clear();
  }
  CK(cudaStreamSynchronize(s.stream));
  return OSAM_OK;
}
}  // namespace
}  // namespace osam

extern "C" {

int osam_set_ic(osam_subdomain* h, const double* u0, const double* v0) {
  if (!h || !u0) return fail(OSAM_EINVAL, "NULL handle or u0");
  Sub& s = h->s;
  if (s.kind == OSAM_ROM && !s.h_phi_rows.empty())
    return fail(OSAM_EINVAL, "ROM with a row subset of Phi cannot restrict a full field: use osam_set_ic_reduced");
  cudaStream_t st = s.stream;
  const size_t nf = (size_t)s.batch * 3 * s.n_nodes;
  double *du = nullptr, *dv = nullptr;
  if (s.kind == OSAM_FOM) {  // stage in the FOM's scratch fields (no allocation per call)
    du = s.scratch_v;
    dv = s.scratch_a;
  } else {
    TRY(dalloc(&du, nf));
    const int rc = dalloc(&dv, nf);
    if (rc != OSAM_OK) {
      dfree(du);
      return rc;
    }
  }
  // copy the caller's fields, then synchronise: the caller's buffers are read only during this call
  cudaError_t e = cudaMemcpyAsync(du, u0, nf * sizeof(double),
                                  is_device_ptr(u0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = v0 == nullptr ? cudaMemsetAsync(dv, 0, nf * sizeof(double), st)
                      : cudaMemcpyAsync(dv, v0, nf * sizeof(double),
                                        is_device_ptr(v0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && s.kind == OSAM_FOM) {
    const int c = s.cur;
    launch_fom_pack(s.g, du, s.st[c][0], s.n_nodes, st);
    launch_fom_pack(s.g, dv, s.st[c][1], s.n_nodes, st);  // RAW state (u, v) until the first osam_step
    g_launches += 2;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    if (s.kind == OSAM_ROM) {
      dfree(du);
      dfree(dv);
    }
    return fail(OSAM_ECUDA, "osam_set_ic copies: %s", cudaGetErrorString(e));
  }
  if (s.kind == OSAM_FOM) {
    s.w_dt = 0.0;
  } else {
    dfree(s.ic_u);
    dfree(s.ic_v);
    dfree(s.ic_s);
    s.ic_u = du;
    s.ic_v = dv;
    s.ic_reduced = false;
  }
  s.ic_pending = true;
  if (s.bound) {
    int launches = 0;
    TRY(process_ic(s, &launches));
    g_launches += launches;
  }
  return OSAM_OK;
}

int osam_set_ic_reduced(osam_subdomain* h, const double* uh0, const double* vh0, const double* s0) {
  if (!h || !uh0) return fail(OSAM_EINVAL, "NULL handle or uh0");
  Sub& s = h->s;
  if (s.kind != OSAM_ROM) return fail(OSAM_EINVAL, "osam_set_ic_reduced applies to a ROM subdomain");
  cudaStream_t st = s.stream;
  const size_t nr = (size_t)s.r * s.batch;
  // the Schwarz DOF count is known only after binding, or from the descriptor's n_s
  const long long ns = s.bound ? s.n_sdof : (s.r_b > 0 ? (long long)(s.h_Phi_s.size() / s.r_b) : -1);
  if (s0 && ns < 0) return fail(OSAM_EINVAL, "s0 given but the Schwarz DOF count is unknown (r_b = 0): bind first");
  double *du = nullptr, *dv = nullptr, *ds = nullptr;
  int rc = dalloc(&du, nr);
  if (rc == OSAM_OK) rc = dalloc(&dv, nr);
  if (rc == OSAM_OK && s0 && ns > 0) rc = dalloc(&ds, (size_t)ns * s.batch);
  cudaError_t e = cudaSuccess;
  if (rc == OSAM_OK) {
    e = cudaMemcpyAsync(du, uh0, nr * sizeof(double),
                        is_device_ptr(uh0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = vh0 == nullptr ? cudaMemsetAsync(dv, 0, nr * sizeof(double), st)
                         : cudaMemcpyAsync(dv, vh0, nr * sizeof(double),
                                           is_device_ptr(vh0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && ds)
      e = cudaMemcpyAsync(ds, s0, sizeof(double) * ns * s.batch,
                          is_device_ptr(s0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(OSAM_ECUDA, "osam_set_ic_reduced copies: %s", cudaGetErrorString(e));
  }
  if (rc != OSAM_OK) {
    dfree(du);
    dfree(dv);
    dfree(ds);
    return rc;
  }
  dfree(s.ic_u);
  dfree(s.ic_v);
  dfree(s.ic_s);
  s.ic_u = du;
  s.ic_v = dv;
  s.ic_s = ds;
  s.ic_reduced = true;
  s.ic_pending = true;
  if (s.bound) {
    int launches = 0;
    TRY(process_ic(s, &launches));
    g_launches += launches;
  }
  return OSAM_OK;
}

int osam_step(osam_subdomain* const* sds, int32_t n_sd, const osam_schwarz_cfg* cfg, int32_t n_steps,
              int32_t* iters_out) {
  if (!sds || n_sd < 1 || !cfg || n_steps < 0) return fail(OSAM_EINVAL, "bad osam_step arguments");
  if (!(cfg->dt > 0) || cfg->max_iters < 1 || cfg->min_iters < 2 || !(cfg->tol_rel >= 0))
    return fail(OSAM_EINVAL, "bad Schwarz configuration (dt > 0, max_iters >= 1, min_iters >= 2)");
  int B = 1;
  for (int i = 0; i < n_sd; ++i) {
    if (!sds[i]) return fail(OSAM_EINVAL, "NULL handle %d", i);
    for (int j = 0; j < i; ++j)
      if (sds[j] == sds[i]) return fail(OSAM_EINVAL, "handle listed twice");
    if (sds[i]->s.stream != sds[0]->s.stream) return fail(OSAM_EINVAL, "all subdomains must share one stream");
    B = std::max(B, sds[i]->s.batch);
  }
  for (int i = 0; i < n_sd; ++i) {
    if (sds[i]->s.batch != B && !(B > 1 && sds[i]->s.batch == B))
      return fail(OSAM_EINVAL, "all subdomains of a batched step must have batch %d (FOMs have batch 1)", B);
  }
  Group* G = nullptr;
  TRY(get_group(sds, n_sd, &G));
  for (int i = 0; i < n_sd; ++i)
    if (sds[i]->s.ic_pending) {
      int launches = 0;
      TRY(process_ic(sds[i]->s, &launches));
      g_launches += launches;
    }
  if (n_steps > 0) {
    int launches = 0;
    for (int i = 0; i < n_sd; ++i) {
      Sub& d = sds[i]->s;
      const double dti = cfg->dt / d.n_sub;
      if (d.kind == OSAM_FOM) TRY(fom_set_step(d, dti, &launches));
      if (d.kind == OSAM_ROM && d.beta > 0.0 && d.minv_dt != dti) {  // (I + beta dt_i^2 e_b Kbar)^-1
        launch_rom_minv(d.r, d.batch, d.Kbar, d.e, d.beta * dti * dti, d.minv_work, d.Minv, d.stream);
        ++launches;
        d.minv_dt = dti;
      }
    }
    g_launches += launches;
  }
  int status = OSAM_OK;
  cudaStream_t st = sds[0]->s.stream;
  if (n_steps > 0) {
    const long long need = (long long)n_steps * B;
    if (need > G->iters_cap) {  // graphs hold the buffer pointer: rebuild them after a reallocation
      for (auto& kv : G->graphs) cudaGraphExecDestroy(kv.second);
      G->graphs.clear();
      dfree(G->iters_all);
      const long long cap = std::max(need, 4096LL * B);
      TRY(dalloc(&G->iters_all, (size_t)cap));
      G->iters_cap = cap;
    }
    // convergence trace (osam_set_conv_trace): graphs hold the buffer pointer, rebuild them on a change
    const long long tneed = g_trace_T > 0 ? (long long)n_steps * g_trace_T * B * 2 : 0;
    if (tneed > G->trace_cap || g_trace_T != G->trace_T) {
      for (auto& kv : G->graphs) cudaGraphExecDestroy(kv.second);
      G->graphs.clear();
      dfree(G->ctrace);
      G->trace_cap = 0;
      G->trace_T = g_trace_T;
      if (tneed > 0) {
        TRY(dalloc(&G->ctrace, (size_t)tneed));
        G->trace_cap = tneed;
      }
    }
    if (G->ctrace) CK(cudaMemsetAsync(G->ctrace, 0xff, sizeof(double) * G->trace_cap, st));  // NaN: not tested
    G->trace_steps = G->ctrace ? n_steps : 0;
    // reset the step counter and the sticky flags of this call
    CK(cudaMemsetAsync(G->ctl_i + 3 + 2 * B, 0, sizeof(int) * 3, st));
  }
  static const bool nograph = getenv("OSAM_NOGRAPH") && getenv("OSAM_NOGRAPH")[0] == '1';
  // small all-FOM groups: one cooperative persistent launch for every step of this call
  bool persist = n_steps > 0 && !g_prof && !nograph && B == 1 && n_sd <= SMALL_MAX_SD && !G->trace &&
                 !(getenv("OSAM_SMALL_PERSIST") && getenv("OSAM_SMALL_PERSIST")[0] == '0');
  for (int i = 0; i < n_sd && persist; ++i) {
    const Sub& d = sds[i]->s;
    persist = d.kind == OSAM_FOM && d.material == OSAM_LINEAR && d.n_sub == 1 && fom_small(d.g) &&
              d.maps.size() <= 6 && d.ux == 1 - d.cur;
  }
  // groups of batched tensor-core ROMs with the folded exchange (c5): one cooperative persistent launch when
  // OSAM_ROM_PERSIST=1 (measured 6.2k vs 6.8k steps/s for the per-step graph on c5: its phases are latency-bound
  // chains of L2 round trips that kernel boundaries do not add much to, so the graph stays the default)
  bool rpersist = n_steps > 0 && !g_prof && !nograph && B > 1 && n_sd <= ROMP_MAX_SD && !G->trace &&
                  getenv("OSAM_ROM_PERSIST") && getenv("OSAM_ROM_PERSIST")[0] == '1';
  for (int i = 0; i < n_sd && rpersist; ++i) {
    const Sub& d = sds[i]->s;
    rpersist = d.kind == OSAM_ROM && d.use_tc && d.fold && d.maps.size() == 1 && d.n_sub == 1 && d.beta == 0.0 &&
               d.nf == 0 && d.batch == B && d.r_b > 0;
  }
  if (rpersist) {
    RomPArgs A{};
    A.n_sd = n_sd;
    A.B = B;
    int slot = 0;
    for (int i = 0; i < n_sd; ++i) {
      Sub& d = sds[i]->s;
      const XferMap& m = d.maps[0];
      RomPSub& p = A.s[i];
      p.r = d.r;
      p.rb = d.r_b;
      p.rz = d.r + d.r_b;
      p.src = m.src;
      p.Gr = sds[m.src]->s.r;
      p.KB = d.KB;
      p.G = m.G;
      p.e = d.e;
      p.Z = d.Z;
      p.part = d.part;
      if (!d.rp_cnt) {
        TRY(dalloc(&d.rp_cnt, (size_t)rom_persist_tiles(d.r, B)));
        CK(cudaMemset(d.rp_cnt, 0, sizeof(int) * rom_persist_tiles(d.r, B)));
      }
      p.cnt = d.rp_cnt;
      for (int b = 0; b < 2; ++b)
        for (int q = 0; q < 4; ++q) p.rst[b][q] = d.rst[b][q];
      p.slot0 = slot;
      slot += rom_persist_slots(d.r);
      p.cur0 = d.cur;
      rom_persist_plan(d.r, d.r_b, p.Gr, B, &p);
    }
    A.n_steps = n_steps;
    A.min_iters = cfg->min_iters;
    A.max_iters = cfg->max_iters;
    A.n_slots = slot;
    A.dt = cfg->dt;
    A.c2 = 0.5 * cfg->dt * cfg->dt;
    A.tol_rel = cfg->tol_rel;
    A.tol_abs = cfg->tol_abs;
    if (!G->ppartial) TRY(dalloc(&G->ppartial, (size_t)slot * B));
    A.partial = G->ppartial;
    A.ctl = G->ctl(cfg->max_iters);
    if (!G->go) TRY(dalloc(&G->go, 1));
    A.go = G->go;
    if (!G->rbar) TRY(dalloc(&G->rbar, 2));
    CK(cudaMemsetAsync(G->rbar, 0, 2 * sizeof(unsigned), st));
    A.bar = G->rbar;
    CK(launch_rom_persistent(A, st));
    ++g_launches;
    if (n_steps & 1)
      for (int i = 0; i < n_sd; ++i) commit_step(sds[i]->s);
  } else if (persist) {
    SmallArgs A{};
    A.n_sd = n_sd;
    int slot = 0;
    for (int i = 0; i < n_sd; ++i) {
      Sub& d = sds[i]->s;
      SmallSub& ss = A.s[i];
      ss.L = fom_launch(d, nullptr, nullptr, nullptr, nullptr, cfg->dt, cfg->dt, 0.5 * cfg->dt, cfg->dt, 0, nullptr,
                        nullptr);
      for (int b = 0; b < 2; ++b)
        for (int q = 0; q < 2; ++q) ss.st[b][q] = d.st[b][q];
      ss.cur0 = d.cur;
      ss.slot0 = slot;
      ss.nvb = fom_slots(d);
      slot += ss.nvb;
      ss.n_maps = (int)d.maps.size();
      for (int k = 0; k < ss.n_maps; ++k) {
        const XferMap& m = d.maps[k];
        ss.maps[k] = SmallMap{m.n, m.src, m.idx, m.out, m.xi};
      }
    }
    A.n_steps = n_steps;
    A.tol_rel = cfg->tol_rel;
    A.tol_abs = cfg->tol_abs;
    A.min_iters = cfg->min_iters;
    A.max_iters = cfg->max_iters;
    A.n_slots = G->n_slots;
    A.partial = G->partial;
    A.ctl = G->ctl(cfg->max_iters);
    if (!G->go) TRY(dalloc(&G->go, 1));
    A.go = G->go;
    const cudaError_t re = launch_small_resident(A, st);
    if (re == cudaErrorNotSupported) {
      cudaGetLastError();
      CK(launch_small_persistent(A, st));
    } else {
      CK(re);
    }
    ++g_launches;
    if (n_steps & 1)
      for (int i = 0; i < n_sd; ++i) commit_step(sds[i]->s);  // the roles alternate every step
  } else if (g_prof || nograph) {
    for (int k = 0; k < n_steps; ++k) {
      const int rc = controller_step_host(*G, *cfg, st);
      if (rc < 0) return rc;
      if (rc == OSAM_WNOTCONVERGED) status = OSAM_WNOTCONVERGED;
    }
  } else {
    for (int k = 0; k < n_steps; ++k) {
      cudaGraphExec_t exec = nullptr;
      int per_sweep = 0;
      TRY(step_graph(*G, *cfg, st, &exec, &per_sweep));
      CK(cudaGraphLaunch(exec, st));
      for (int i = 0; i < n_sd; ++i) commit_step(sds[i]->s);  // commit (buffer roles)
    }
  }
  std::vector<int32_t> its;
  if (n_steps > 0) {
    its.resize((size_t)n_steps * B);
    CK(cudaMemcpyAsync(G->h_ctl, G->ctl_i, sizeof(int) * G->ctl_len(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(its.data(), G->iters_all, sizeof(int32_t) * its.size(), cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (n_steps > 0) {
    if (iters_out) std::memcpy(iters_out, its.data(), sizeof(int32_t) * its.size());
    if (!(g_prof || nograph) && !persist && !rpersist) {  // kernels the graphs ran: step_begin + the sweeps (max over samples)
      for (int k = 0; k < n_steps; ++k) {
        int nmax = 0;
        for (int b = 0; b < B; ++b) nmax = std::max(nmax, its[(size_t)k * B + b]);
        g_launches += G->launches_begin + (long long)nmax * G->launches_per_sweep;
      }
    }
    if (G->h_ctl[4 + 2 * B]) return fail(OSAM_EUNSTABLE, "non-finite Schwarz convergence norm");
    if (G->h_ctl[5 + 2 * B]) status = OSAM_WNOTCONVERGED;
  }
  return status;
}

static int copy_out(const double* src, double* dst, size_t n, cudaStream_t st) {
  if (is_device_ptr(dst))
    CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  else
    CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  return OSAM_OK;
}

static int get_field(const osam_subdomain* h, int which, double* out) {
  const Sub& s = h->s;
  if (s.ic_pending) return fail(OSAM_EINVAL, "initial condition not processed yet: call osam_step first");
  cudaStream_t st = s.stream;
  if (s.kind == OSAM_FOM) {
    const double* field = s.st[s.w_dt == 0.0 ? s.cur : s.ux][0];  // u (R30)
    if (which != 0) {
      // a = -K u / m and v = w - w_dt/2 a by one force pass into the spare buffer (the committed
      // state is not modified).
      if (!s.bound) return fail(OSAM_EINVAL, "FOM state not bound: call osam_step first");
      int launches = 0;
      const int xb = s.w_dt == 0.0 ? s.cur : s.ux;  // buffer holding u
      const FomLaunch L = fom_launch(s, s.st[xb][0], s.st[s.cur][1], nullptr, s.scratch_v, -0.5 * s.w_dt, 0.0, 0.0,
                                     0.0, 0, s.scratch_partial, s.scratch_a);
      launch_fom_advance(L, s.stencil, &s.tmap[xb], &s.tmapw[s.cur], &s.tmapw[s.cur], st, &launches);
      g_launches += launches;
      field = which == 1 ? s.scratch_v : s.scratch_a;
    }
    double* tmp = which == 2 ? s.scratch_v : s.scratch_a;  // not the source field
    launch_fom_unpack(s.g, field, tmp, s.n_nodes, st);
    ++g_launches;
    const int rc = copy_out(tmp, out, (size_t)3 * s.n_nodes, st);
    CK(cudaStreamSynchronize(st));
    return rc;
  }
  if (!s.bound) return fail(OSAM_EINVAL, "ROM state not initialised: call osam_step first");
  TRY(copy_out(s.rst[s.cur][which], out, (size_t)s.r * s.batch, st));
  CK(cudaStreamSynchronize(st));
  return OSAM_OK;
}

int osam_get_state(const osam_subdomain* h, double* u_out, double* v_out) {
  if (!h) return fail(OSAM_EINVAL, "NULL handle");
  if (u_out) TRY(get_field(h, 0, u_out));
  if (v_out) TRY(get_field(h, 1, v_out));
  return OSAM_OK;
}

int osam_get_accel(const osam_subdomain* h, double* a_out) {
  if (!h || !a_out) return fail(OSAM_EINVAL, "NULL argument");
  return get_field(h, 2, a_out);
}

int osam_get_sizes(const osam_subdomain* h, int64_t* n_nodes, int64_t* n_free, int64_t* n_schwarz, int32_t* batch) {
  if (!h) return fail(OSAM_EINVAL, "NULL handle");
  if (n_nodes) *n_nodes = h->s.n_nodes;
  if (n_free) *n_free = h->s.bound ? h->s.n_free : -1;
  if (n_schwarz) *n_schwarz = h->s.bound ? h->s.n_sdof : -1;
  if (batch) *batch = h->s.batch;
  return OSAM_OK;
}

void osam_destroy(osam_subdomain* h) {
  if (!h) return;
  forget_groups_with(h);
  Sub& s = h->s;
  if (s.stream) cudaStreamSynchronize(s.stream);
  release_binding(s);
  for (int b = 0; b < 3; ++b)
    for (int q = 0; q < 2; ++q) dfree(s.st[b][q]);
  dfree(s.zbuf);
  dfree(s.scratch_a);
  dfree(s.scratch_v);
  dfree(s.coef);
  dfree(s.rowc);
  dfree(s.ic_u);
  dfree(s.ic_v);
  dfree(s.ic_s);
  delete h;
}

int osam_opinf_replay(const osam_replay_desc* d, double* err_out, int32_t* best_out, double* traj_out,
                      void* cuda_stream) {
  if (!d || !err_out) return fail(OSAM_EINVAL, "NULL descriptor or err_out");
  if (d->r < 1 || d->r_b < 0 || d->n_models < 1 || d->n_steps < 1 || d->order < 1 || d->order > 3 || !(d->dt > 0))
    return fail(OSAM_EINVAL, "replay needs r >= 1, r_b >= 0, n_models >= 1, n_steps >= 1, order 1..3, dt > 0");
  if (!d->O || !d->Ubar || (d->r_b > 0 && !d->Ghat)) return fail(OSAM_EINVAL, "replay input pointer is NULL");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const long long r = d->r, rb = d->r_b, K = d->n_steps, B = d->n_models;
  const long long n2 = d->order >= 2 ? r * (r + 1) / 2 : 0, n3 = d->order >= 3 ? r * (r + 1) * (r + 2) / 6 : 0;
  const long long nf = n2 + n3, rz = r + rb + nf;
  std::vector<int> idx;
  for (int i = 0; i < r && d->order >= 2; ++i)
    for (int j = i; j < r; ++j) idx.insert(idx.end(), {i, j, -1});
  for (int i = 0; i < r && d->order >= 3; ++i)
    for (int j = i; j < r; ++j)
      for (int l = j; l < r; ++l) idx.insert(idx.end(), {i, j, l});
  // device copies (per call: an offline routine)
  double *O_cm = nullptr, *O = nullptr, *Ub = nullptr, *Gh = nullptr, *v0 = nullptr, *z = nullptr, *err = nullptr,
         *traj = nullptr;
  int *fi = nullptr, *best = nullptr;
  int rc = OSAM_OK;
  auto in = [&](double** dst, const double* src, long long n) -> int {
    TRY(dalloc_async(dst, (size_t)std::max(1LL, n), st));
    if (n > 0)
      CK(cudaMemcpyAsync(*dst, src, sizeof(double) * n,
                         is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    return OSAM_OK;
  };
  do {
    if ((rc = in(&O_cm, d->O, B * r * rz)) != OSAM_OK) break;
    if ((rc = dalloc_async(&O, (size_t)(B * r * rz), st)) != OSAM_OK) break;
    if ((rc = in(&Ub, d->Ubar, r * K)) != OSAM_OK) break;
    if ((rc = in(&Gh, d->Ghat, rb * K)) != OSAM_OK) break;
    if (d->vh0 && (rc = in(&v0, d->vh0, r)) != OSAM_OK) break;
    if ((rc = dalloc_async(&z, (size_t)(B * rz), st)) != OSAM_OK) break;
    if ((rc = dalloc_async(&err, (size_t)B, st)) != OSAM_OK) break;
    if ((rc = dalloc_async(&best, 1, st)) != OSAM_OK) break;
    if (traj_out && (rc = dalloc_async(&traj, (size_t)(B * K * r), st)) != OSAM_OK) break;
    if (!idx.empty()) {
      if ((rc = dalloc_async(&fi, idx.size(), st)) != OSAM_OK) break;
      const cudaError_t e = cudaMemcpyAsync(fi, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) {
        rc = fail(OSAM_ECUDA, "replay: %s", cudaGetErrorString(e));
        break;
      }
    }
    launch_transpose_ops((int)r, (int)rz, (int)B, O_cm, O, st);
    ReplayArgs A{};
    A.r = (int)r;
    A.r_b = (int)rb;
    A.nf = (int)nf;
    A.B = (int)B;
    A.K = (int)K;
    A.dt = d->dt;
    A.O = O;
    A.feat_idx = fi;
    A.Ubar = Ub;
    A.Ghat = Gh;
    A.vh0 = v0;
    A.z = z;
    A.traj = traj;
    A.err = err;
    A.best = best;
    cudaError_t e = launch_replay(A, st);
    if (e != cudaSuccess) {
      rc = fail(OSAM_ECUDA, "replay launch: %s", cudaGetErrorString(e));
      break;
    }
    g_launches += 3;
    if ((rc = copy_out(err, err_out, (size_t)B, st)) != OSAM_OK) break;
    if (traj_out && (rc = copy_out(traj, traj_out, (size_t)(B * K * r), st)) != OSAM_OK) break;
    int hb = -1;
    e = cudaMemcpyAsync(&hb, best, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      rc = fail(OSAM_ECUDA, "replay: %s", cudaGetErrorString(e));
      break;
    }
    if (best_out) *best_out = hb;
  } while (false);
  dfree_async(O_cm, st);
  dfree_async(O, st);
  dfree_async(Ub, st);
  dfree_async(Gh, st);
  dfree_async(v0, st);
  dfree_async(z, st);
  dfree_async(err, st);
  dfree_async(best, st);
  dfree_async(traj, st);
  dfree_async(fi, st);
  cudaStreamSynchronize(st);  // the idx host vector and the caller's outputs must outlive the copies
  return rc;
}

void osam_set_profiling(int32_t on) { g_prof = on != 0; }

void osam_set_conv_trace(int32_t max_n) { g_trace_T = max_n > 0 ? max_n : 0; }

int osam_get_k1_timeline(osam_subdomain* const* sds, int32_t n_sd, int32_t reset, double* out) {
  if (!sds || n_sd < 1 || !out) return fail(OSAM_EINVAL, "bad osam_get_k1_timeline arguments");
  auto it = g_groups.find(std::vector<osam_subdomain*>(sds, sds + n_sd));
  if (it == g_groups.end()) return fail(OSAM_EINVAL, "no osam_step call on this subdomain list");
  const Group& G = *it->second;
  cudaStream_t st = sds[0]->s.stream;
  double b[5];
  CK(cudaMemcpyAsync(b, G.busy, sizeof b, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double base = 0.0, band = 0.0;  // algorithmic bytes per sweep (R38) of the timed K1s
  for (auto h : G.sds) {
    const Sub& d = h->s;
    if (d.kind != OSAM_FOM || d.material != OSAM_LINEAR || d.n_sub != 1 || fom_small(d.g)) continue;
    base += 32.0 * 3.0 * (double)d.n_nodes;
    band += 8.0 * 3.0 * (double)d.n_band;
  }
  out[0] = b[0] * 1e-6;
  out[1] = b[1] * 1e-6;
  out[2] = b[2];
  out[3] = b[3];
  out[4] = b[4];
  out[5] = b[3] * base + b[4] * band;
  if (reset) {
    CK(cudaMemsetAsync(G.busy, 0, sizeof(double) * 5, st));
    CK(cudaStreamSynchronize(st));
  }
  return OSAM_OK;
}

int osam_get_conv_trace(osam_subdomain* const* sds, int32_t n_sd, double* out, int32_t* n_steps, int32_t* max_n,
                        int32_t* batch) {
  if (!sds || n_sd < 1) return fail(OSAM_EINVAL, "bad osam_get_conv_trace arguments");
  auto it = g_groups.find(std::vector<osam_subdomain*>(sds, sds + n_sd));
  if (it == g_groups.end()) return fail(OSAM_EINVAL, "no osam_step call on this subdomain list");
  const Group& G = *it->second;
  if (n_steps) *n_steps = G.trace_steps;
  if (max_n) *max_n = G.trace_T;
  if (batch) *batch = G.B;
  if (out && G.ctrace && G.trace_steps > 0) {
    cudaStream_t st = sds[0]->s.stream;
    TRY(copy_out(G.ctrace, out, (size_t)G.trace_steps * G.trace_T * G.B * 2, st));
    CK(cudaStreamSynchronize(st));
  }
  return OSAM_OK;
}

void osam_reset_profile(void) {
  g_k1_ms = 0.0;
  g_k1_launches = 0;
  g_k1_bytes = 0.0;
  g_launches = 0;
}

void osam_get_profile(double* k1_ms, int64_t* k1_launches, double* k1_bytes, int64_t* kernel_launches) {
  if (k1_ms) *k1_ms = g_k1_ms;
  if (k1_launches) *k1_launches = g_k1_launches;
  if (k1_bytes) *k1_bytes = g_k1_bytes;
  if (kernel_launches) *kernel_launches = g_launches;
}

}  // extern "C"
