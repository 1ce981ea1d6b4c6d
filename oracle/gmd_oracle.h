/* ORACLE TEST INFRASTRUCTURE -- not part of the product.
 *
 * Plain-C, fp64 restatement of the reference graphmd hot path
 * (/root/reference/proj/src/{system,neighborlist,partitioner,linegraph,
 * potential}.cpp).  Used only by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py, as the checker.  Pinned against the compiled
 * reference (oracle/_ref) and tests/golden/ by tests/test_oracle.py.
 *
 * Conventions: positions/vectors are row-major N x 3 doubles, the lattice is
 * 3 x 3 row-major with rows = cell vectors, image offsets are int32 triples.
 * Every function returns 0 on success and nonzero on error, with the message
 * available from orc_last_error() (same text as the reference's Error).
 */
#ifndef GMD_ORACLE_H
#define GMD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* deterministic RNG: mt19937_64 + Box-Muller (system.hpp:121-149) */
void orc_rng_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out);
void orc_rng_normal(uint64_t seed, int64_t count, double* out);

/* make_supercell + random_perturb (system.cpp:188-240); amp <= 0 skips */
void orc_supercell(int64_t n, const double* pos, const int32_t* z, const double* lat,
                   int rx, int ry, int rz, double amp, uint64_t seed,
                   double* out_pos, int32_t* out_z, double* out_lat);

/* ToyPotentialParams::init (potential.cpp:119-148) into the flat blob:
 * emb[119F] | layer_w[LFF] | layer_b[LF] | basis_proj[FK] | basis3_proj[FK] |
 * w3[FF] | w4[FF] | readout[F] */
int64_t orc_params_size(int F, int K, int L);
void orc_params_init(uint64_t seed, int F, int K, int L, double r_atom, double r3,
                     double* blob);

/* ---- neighbour list (neighborlist.cpp:108-239) ---- */
void* orc_neighbor_list(int64_t n, const double* pos, const int32_t* z,
                        const double* lat, const uint8_t* pbc, double rc, int brute);
int64_t orc_graph_num_edges(void* g);
void orc_graph_get(void* g, int64_t* src, int64_t* dst, int32_t* off, double* dist,
                   double* vec);
void orc_graph_destroy(void* g);

/* ---- Distributed::create_distributed equivalent (engine.cpp:44-65) ---- */
void* orc_create(int64_t n, const double* pos, const int32_t* z, const double* lat,
                 const uint8_t* pbc, double rc, double r3, double tau, int p,
                 int allow_narrow);
void orc_destroy(void* h);
int64_t orc_num_nodes(void* h);
int64_t orc_num_edges(void* h);
void orc_graph(void* h, int64_t* src, int64_t* dst, int32_t* off, double* dist,
               double* vec);
void orc_system(void* h, double* pos, double* lat);
int orc_rule(void* h, double* boundaries);
void orc_owner(void* h, int32_t* owner);
int64_t orc_layout_size(void* h, int part, int bonds);
void orc_layout(void* h, int part, int bonds, int64_t* node_array, int64_t* markers);
int64_t orc_num_dups(void* h, int part, int bonds);
void orc_dups(void* h, int part, int bonds, int64_t* pairs);
int64_t orc_num_owned_edges(void* h, int part);
void orc_owned_edges(void* h, int part, int64_t* owned, int64_t* lsrc, int64_t* ldst);
int64_t orc_num_border(void* h, int part);
void orc_border(void* h, int part, int64_t* out);
int orc_has_line_graph(void* h);
int64_t orc_num_bonds(void* h);
void orc_bonds(void* h, int64_t* edge_of_bond, int32_t* bond_owner);
int64_t orc_num_line_edges(void* h, int part);
void orc_line_edges(void* h, int part, int64_t* pairs);

/* serial (brute=0, linegraph.cpp:183-200) or brute-force (brute=1,
 * :202-219) global line graph as sorted (edge e, edge e') pairs */
void* orc_line_graph(int64_t n, const double* pos, const int32_t* z, const double* lat,
                     const uint8_t* pbc, double rc, double r, double tau, int brute);
int64_t orc_pairs_size(void* ph);
void orc_pairs_get(void* ph, int64_t* out);
void orc_pairs_destroy(void* ph);

/* ---- forward_serial (potential.cpp:269-530) ---- */
int orc_forward_serial(int64_t n, const double* pos, const int32_t* z, const double* lat,
                       const uint8_t* pbc, int F, int K, int L, double r_atom, double r3,
                       const double* blob, double* energy, double* per_atom,
                       double* forces, double* stress);

/* ---- MD (md.cpp:11-160) ---- */
double orc_atomic_mass(int z);
/* init_md_state + forces at pos0, then `steps` velocity-Verlet steps; final
 * pos / vel / forces (n x 3) and records rec[(steps + 1) x 4] = (potential,
 * kinetic, total, max |f|) per step, row 0 = initial */
int orc_md_run(int64_t n, const double* pos0, const int32_t* z, const double* lat,
               const uint8_t* pbc, int F, int K, int L, double r_atom, double r3,
               const double* blob, double dt, int64_t steps, double temperature, uint64_t seed,
               double* pos, double* vel, double* forces, double* rec);

#ifdef __cplusplus
}
#endif
#endif
