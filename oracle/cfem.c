/*
 * Oracle: hex8 element-loop internal force in plain C (TEST INFRASTRUCTURE ONLY, see
 * oracle/__init__.py; loaded by oracle/cfem.py, never by the product path).
 *
 * The same definition as oracle/fem.py internal_force (P:L133-137 eq:matrix_vector_form,
 * SURVEY 8(c) c.1 step 4):
 *
 *     f = sum over elements e of scatter( K_e u_e ),
 *
 * K_e the 24 x 24 element stiffness (computed by oracle/fem.py hex8_stiffness with 2x2x2 Gauss
 * points and passed in, row/column order (local node a, component c) -> 3a + c), u_e the 24
 * displacements of the element's nodes in the local order (---, +--, ++-, -+-, --+, +-+, +++, -++).
 * Written as a plain element loop for the large configurations (c3, c4, c4 training) where the
 * NumPy loop takes seconds per evaluation.  Parallelised with the 8-colouring of SURVEY 7 step 0:
 * elements of one colour (ei%2, ej%2, ek%2) share no node, so every node receives its (up to 8)
 * element contributions in colour order whatever the thread count -> deterministic.
 * Node id p = i + (nx+1)(j + (ny+1)k); arrays node-major (n_nodes, 3).
 */
#include <omp.h>
#include <stdint.h>
#include <string.h>

/* thread count of the element loop (timing of the oracle baseline at 1 thread and at all cores) */
void oracle_set_threads(int32_t n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
int32_t oracle_get_threads(void) { return omp_get_max_threads(); }

static const int LOC[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                              {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

void oracle_internal_force(int32_t nx, int32_t ny, int32_t nz, const double* Ke, const double* u,
                           double* f) {
  const int64_t px = nx + 1, py = ny + 1;
  const int64_t n_nodes = px * py * (int64_t)(nz + 1);
  memset(f, 0, sizeof(double) * 3 * (size_t)n_nodes);
  for (int colour = 0; colour < 8; ++colour) {
    const int ci = colour & 1, cj = (colour >> 1) & 1, ck = (colour >> 2) & 1;
#pragma omp parallel for collapse(2) schedule(static)
    for (int32_t ek = ck; ek < nz; ek += 2) {
      for (int32_t ej = cj; ej < ny; ej += 2) {
        for (int32_t ei = ci; ei < nx; ei += 2) {
          int64_t node[8];
          double ue[24], fe[24];
          for (int a = 0; a < 8; ++a) {
            node[a] = (ei + LOC[a][0]) + px * ((ej + LOC[a][1]) + py * (int64_t)(ek + LOC[a][2]));
            for (int c = 0; c < 3; ++c) ue[3 * a + c] = u[3 * node[a] + c];
          }
          for (int row = 0; row < 24; ++row) {
            double acc = 0.0;
            for (int col = 0; col < 24; ++col) acc += Ke[24 * row + col] * ue[col];
            fe[row] = acc;
          }
          for (int a = 0; a < 8; ++a)
            for (int c = 0; c < 3; ++c) f[3 * node[a] + c] += fe[3 * a + c];
        }
      }
    }
  }
}
