/*
 * graphmd_b200 -- C ABI of the B200-native graph-partitioned MLIP inference
 * path (DistMLIP -> graphmd).  Drop-in for the reference's plugin API:
 *
 *   graphmd::Distributed::create_distributed   proj/include/graphmd/engine.hpp:51-56
 *   graphmd::forward_distributed               proj/include/graphmd/potential.hpp:58-60
 *   Distributed feature API (transfer, transpose, duplicates, distribute,
 *   aggregate)                                 proj/include/graphmd/engine.hpp:74-129
 *   graph / partition / line-graph views       engine.hpp:58-72, neighborlist.hpp:17-33,
 *                                              partitioner.hpp:16-82, linegraph.hpp:15-54
 *
 * Plain C types only.  Every function returns GMD_OK (0) or an error code;
 * the message (same text as the reference's graphmd::Error where one exists)
 * is available from gmd_last_error(h).  Host pointers unless a flag says
 * otherwise.  One control thread per handle (SPEC: one thread drives the API).
 *
 * Buffers: the handle owns all device memory, grows it on demand and reuses
 * it across builds (per-MD-step rebuilds do not reallocate).
 */
#ifndef GRAPHMD_B200_H
#define GRAPHMD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GMD_OK 0
#define GMD_ERR_CONFIG 2  /* invalid input/configuration (reference: Error) */
#define GMD_ERR_RUNTIME 3 /* runtime failure: non-finite feature, plan misalignment */
#define GMD_ERR_CUDA 4    /* CUDA / NCCL failure */
#define GMD_ERR_ARG 5     /* bad handle / null pointer / index out of range */

/* gmd_build flags */
#define GMD_ALLOW_NARROW 1u   /* allow slabs narrower than the cutoff (partitioner.cpp:21-33) */
#define GMD_INPUT_DEVICE 2u   /* pos/Z are device pointers on the handle's GPU */
#define GMD_EQUAL_WIDTH 4u    /* BoundaryMode::kEqualWidth (partitioner.hpp:22-25) */
#define GMD_LINE_PARTS 8u     /* build the per-partition line-graph edges inside gmd_build, as
                                 create_distributed does (engine.cpp:57-62); the model does not
                                 need them, the views build them on first use otherwise */

/* gmd_forward flags */
#define GMD_OUTPUT_DEVICE 1u  /* output pointers are device pointers */
#define GMD_OUTPUT_F32 2u     /* per_atom / forces are float instead of double */

/* feature dtypes; OR GMD_HOST_MEMORY into dtype when the feature buffer of a
 * feature-API call is host memory (it is staged through device scratch) */
#define GMD_F32 0
#define GMD_F64 1
#define GMD_HOST_MEMORY 0x100

typedef struct gmd_handle gmd_handle;

const char* gmd_version(void);
const char* gmd_last_error(const gmd_handle* h);

/* one handle per process and GPU (device ordinal) */
int gmd_create(int device, gmd_handle** out);
void gmd_destroy(gmd_handle* h);

/* Distributed::create_distributed(system, atom_cutoff, threebody_cutoff, p,
 * n_threads, allow_narrow, threebody_tau) -- engine.hpp:51-56.
 * pos: n x 3 Cartesian (A), Z: n atomic numbers, lattice: 3 x 3 rows,
 * pbc: 3 flags (NULL = fully periodic), r3 <= 0 disables the line graph.
 * n_threads is accepted and ignored (the GPU path is deterministic). */
int gmd_build(gmd_handle* h, int64_t n, const double* pos, const int32_t* Z,
              const double lattice[9], const uint8_t pbc[3], double rc, double r3,
              double tau, int p, int n_threads, uint32_t flags);

/* ToyPotentialParams (potential.hpp:15-41) as a flat fp64 blob:
 * emb[119F] | layer_w[LFF] | layer_b[LF] | basis_proj[FK] | basis3_proj[FK] |
 * w3[FF] | w4[FF] | readout[F].  The compiled kernels support F=16, K=8, L<=8. */
int gmd_set_params(gmd_handle* h, int F, int K, int L, double r_atom, double r3,
                   const double* blob);
/* ToyPotentialParams::init (potential.cpp:119-148), host-side */
int64_t gmd_params_size(int F, int K, int L);
int gmd_params_init(uint64_t seed, int F, int K, int L, double r_atom, double r3,
                    double* blob);

/* forward_distributed(dist, params, timing) -- potential.hpp:58-60.
 * energy (1), per_atom (n), forces (n x 3), stress (9, row-major), timing (4:
 * graph creation of the last build, feature calc, forward, backward; seconds).
 * Any output pointer may be NULL. */
int gmd_forward(gmd_handle* h, double* energy, void* per_atom, void* forces, double* stress,
                double* timing, uint32_t flags);

/* ---- on-device MD: the caller of the hot path (md.hpp:49-89, md.cpp) ------
 * State arrays are DEVICE pointers on the handle's GPU, fp64: pos, vel,
 * forces (n x 3), masses (n); Z (n int32, device).  gmd_set_params first. */
/* atomic_mass(Z) (system.cpp:289-293), host arrays */
int gmd_md_masses(int64_t n, const int32_t* Z, double* masses);
/* maxwell_boltzmann_velocities(system, T, seed) (md.cpp:20-52), host arrays */
int gmd_md_maxwell_boltzmann(int64_t n, const int32_t* Z, double temperature, uint64_t seed,
                             double* vel);
/* evaluate (md.cpp:55-69): rebuild graph + partitions at pos, forward, forces
 * (device) <- -dE/dr; energy (host) and timing (4, host) optional */
int gmd_md_evaluate(gmd_handle* h, int64_t n, const double* pos, const int32_t* Z,
                    const double lattice[9], const uint8_t pbc[3], double rc, double r3, double tau,
                    int p, uint32_t flags, double* forces, double* energy, double* timing);
/* velocity_verlet_step (md.cpp:85-110): half-kick + drift, wrap_positions,
 * evaluate, half-kick; forces must hold the forces at pos on entry.  A
 * non-finite force fails with GMD_ERR_RUNTIME ("non-finite force on atom i"). */
int gmd_md_step(gmd_handle* h, int64_t n, double* pos, double* vel, double* forces,
                const double* masses, const int32_t* Z, const double lattice[9],
                const uint8_t pbc[3], double dt, double rc, double r3, double tau, int p,
                uint32_t flags, double* energy, double* timing);
/* MDState::kinetic_energy (eV) and max |f| (eV/A) of the device state; forces
 * may be NULL */
int gmd_md_observe(gmd_handle* h, int64_t n, const double* vel, const double* masses,
                   const double* forces, double* kinetic, double* max_force);

/* run_md (md.cpp:112-160) with HOST state in/out and the whole trajectory on
 * the device: evaluate at pos, then `steps` velocity-Verlet steps.  pos / vel
 * (n x 3) are read and overwritten with the final state, forces (optional)
 * receives the final forces; records (optional, (steps + 1) x 8) holds per
 * step: potential, kinetic, total, max |f|, graph creation, feature calc,
 * forward, backward (s). */
int gmd_md_run(gmd_handle* h, int64_t n, double* pos, double* vel, double* forces,
               const int32_t* Z, const double lattice[9], const uint8_t pbc[3], double dt,
               int64_t steps, double rc, double r3, double tau, int p, uint32_t flags,
               double* records);

/* ---- views (parity / export; materialized on demand) -------------------- */
int gmd_num_nodes(const gmd_handle* h, int64_t* n);
int gmd_num_edges(const gmd_handle* h, int64_t* ne);
int gmd_num_partitions(const gmd_handle* h, int* p);
/* AtomGraph in canonical order; off = image_offset (n x 3 int32) */
int gmd_get_graph(gmd_handle* h, int64_t* src, int64_t* dst, int32_t* off, double* dist,
                  double* vec);
/* ensure_periodic (system.cpp:242-270) on the device: non-periodic axes padded
 * to extent + 2 cutoff, positions shifted by cutoff - lo */
int gmd_util_ensure_periodic(gmd_handle* h, int64_t n, const double* pos, const double lattice[9],
                             const uint8_t pbc[3], double cutoff, double* out_pos, double* out_lat);
/* canonical CSR by destination: row (n + 1), src (ne), int32 */
int gmd_get_csr(gmd_handle* h, int32_t* row, int32_t* src);
/* system after ensure_periodic (positions n x 3, lattice 3 x 3) */
int gmd_get_system(gmd_handle* h, double* pos, double* lattice);
/* PartitionRule: axis and p + 1 boundaries */
int gmd_get_rule(gmd_handle* h, int* axis, double* boundaries);
int gmd_get_owner(gmd_handle* h, int32_t* owner);
/* SpanLayout of partition `part` over atoms (bonds = 0) or bonds (bonds = 1) */
int gmd_get_layout_size(gmd_handle* h, int part, int bonds, int64_t* size);
int gmd_get_layout(gmd_handle* h, int part, int bonds, int64_t* node_array,
                   int64_t* markers /* 2 + 2p */);
int gmd_get_num_duplicates(gmd_handle* h, int part, int bonds, int64_t* count);
int gmd_get_duplicates(gmd_handle* h, int part, int bonds, int64_t* pairs);
/* AtomPartition: owned edges (ascending global id) and canonical local ends */
int gmd_get_num_owned_edges(gmd_handle* h, int part, int64_t* count);
int gmd_get_owned_edges(gmd_handle* h, int part, int64_t* owned, int64_t* local_src,
                        int64_t* local_dst);
int gmd_get_num_border_edges(gmd_handle* h, int part, int64_t* count);
int gmd_get_border_edges(gmd_handle* h, int part, int64_t* border);
/* PartitionedLineGraph */
int gmd_has_line_graph(const gmd_handle* h, int* yes);
int gmd_get_num_bonds(gmd_handle* h, int64_t* nb);
int gmd_get_bonds(gmd_handle* h, int64_t* edge_of_bond, int32_t* bond_owner);
int gmd_get_num_line_edges(gmd_handle* h, int part, int64_t* count);
int gmd_get_line_edges(gmd_handle* h, int part, int64_t* pairs /* (local e, local e') */);

/* ---- free builders (device-backed) ---------------------------------------
 * The reference's public lower-level builders on the GPU; every view getter
 * above then reads the handle.  Replaces, one for one:
 *   choose_partition_rule  partitioner.hpp:91-92 / partitioner.cpp:46-91
 *   fractional_along_axis, which_partition(node)  partitioner.hpp:94-99
 *   assign_to_partitions, build_atom_partitions  partitioner.hpp:101-109
 *   build_two_hop_closure  linegraph.hpp:58-59
 *   build_edge_tables (per-partition table membership)  linegraph.hpp:61-64
 *   build_line_graph_partitions, serial_line_graph  linegraph.hpp:66-73
 *   brute_force_line_graph  linegraph.hpp:75-78
 *   brute_force_neighbor_list  neighborlist.hpp:40-42 */
/* choose_partition_rule: axis = longest lattice row; p + 1 boundaries
 * (quantile walls by a device radix select, or equal widths) */
int gmd_partition_rule(gmd_handle* h, int64_t n, const double* pos, const double lattice[9], int p,
                       int equal_width, int* axis, double* boundaries);
/* wrapped fractional coordinate along `axis` (fracs, may be NULL) and
 * which_partition of every atom (owner, may be NULL; needs the rule) */
int gmd_assign_owners(gmd_handle* h, int64_t n, const double* pos, const double lattice[9], int axis,
                      int p, const double* boundaries, double* fracs, int32_t* owner);
/* partitions (+ bonds / line graph when r3 > 0) of a caller-supplied graph in
 * canonical dst-major order; owners from `owner` if non-NULL, else from
 * positions + rule.  flags: GMD_ALLOW_NARROW.  The handle then serves the
 * partition / bond / line-graph getters and the feature API (no forward). */
int gmd_build_partitions(gmd_handle* h, int64_t n, const double* pos, const double lattice[9],
                         int64_t ne, const int64_t* src, const int64_t* dst, const int32_t* off,
                         const double* dist, double cutoff, double r3, double tau, int axis, int p,
                         const double* boundaries, const int32_t* owner, uint32_t flags);
/* two-hop closure of partition `part`: ascending node ids (ids may be NULL) */
int gmd_get_closure(gmd_handle* h, int part, int64_t* count, int64_t* ids);
/* edge-table membership: bit i of mask[b] = bond b in partition i's table */
int gmd_get_bond_tables(gmd_handle* h, uint64_t* mask);
/* brute-force line graph of the handle's bonds: sorted (edge e, edge e') */
int gmd_brute_force_line_graph(gmd_handle* h, int64_t* count, int64_t* pairs);
/* brute-force radius graph (N <= 5000), canonical order; with all output
 * pointers NULL only *ne is returned */
int gmd_brute_force_neighbor_list(gmd_handle* h, int64_t n, const double* pos,
                                  const double lattice[9], const uint8_t pbc[3], double cutoff,
                                  int64_t* ne, int64_t* src, int64_t* dst, int32_t* off,
                                  double* dist, double* vec);

/* ---- Distributed feature API (engine.hpp:74-129) -------------------------
 * Per-partition blocks live in ONE device buffer: partition i's block starts
 * at row gmd_block_offset(i) and has layout-size rows of `width` elements. */
int gmd_block_rows(gmd_handle* h, int bonds, int64_t* total_rows);
int gmd_block_offset(gmd_handle* h, int part, int bonds, int64_t* row0);
int gmd_transfer(gmd_handle* h, int bonds, void* dev_buf, int width, int dtype);
int gmd_transfer_transpose(gmd_handle* h, int bonds, void* dev_buf, int width, int dtype);
int gmd_sync_duplicates(gmd_handle* h, int bonds, void* dev_buf, int width, int dtype);
/* host global [rows x width] <-> device blocks */
int gmd_distribute(gmd_handle* h, int bonds, const void* host_global, void* dev_buf, int width,
                   int dtype);
int gmd_aggregate(gmd_handle* h, int bonds, const void* dev_buf, void* host_global, int width,
                  int dtype);
/* negative-control hook (engine.cpp:296): corrupt one transfer plan entry */
int gmd_corrupt_transfer_plan_for_test(gmd_handle* h);

/* ---- one rank per GPU ----------------------------------------
 * Rank r of `world` owns slab r of p = world partitions: gmd_build then builds
 * only r's rows (positions are replicated inputs), and gmd_forward exchanges
 * halo rows with the peers every layer.  Outputs (per_atom, forces) are
 * written for r's atoms only (zeros elsewhere); energy and stress are global.
 * Transports: NCCL (one process per GPU; rank 0 makes the id, the caller
 * broadcasts it) or an in-process group of handles (each driven by its own
 * host thread; device-to-device copies). */
int gmd_comm_nccl_id(uint8_t id[128]);
int gmd_comm_init_nccl(gmd_handle* h, int rank, int world, const uint8_t id[128]);
int gmd_comm_init_local(gmd_handle** handles, int world);
/* CUDA-IPC peer transport for ranks on one node (one process per GPU, or
 * several processes sharing a GPU): the halo rows of every exchange are
 * stored straight into the receiving rank's window (P2P over NVLink), with
 * stream-ordered flag handshakes -- no NCCL, no host round trip.
 * 1. gmd_comm_ipc_export: allocate this rank's window (slot_rows rows of 16
 *    floats per peer, double-buffered) and get its 64-byte IPC handle;
 * 2. all-gather the handles (rank order) over any host channel;
 * 3. gmd_comm_init_ipc(h, handles[world x 64]) before gmd_build. */
int gmd_comm_ipc_export(gmd_handle* h, int rank, int world, int64_t slot_rows,
                        uint8_t handle[64]);
int gmd_comm_init_ipc(gmd_handle* h, const uint8_t* handles);
int gmd_comm_info(const gmd_handle* h, int* rank, int* world);
int gmd_num_owned(const gmd_handle* h, int64_t* n);
int gmd_get_owned_ids(gmd_handle* h, int64_t* ids);
/* owned atoms with no in-edge from a peer's atom: their layer updates run
 * while the halo exchange is in flight (GMD_OVERLAP=0 disables the split) */
int gmd_num_interior(const gmd_handle* h, int64_t* n);

/* ---- input synthesis helpers (system.hpp:99-149; host-side) ------------- */
int gmd_util_rng_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out);
int gmd_util_supercell(int64_t n, const double* pos, const int32_t* Z, const double lattice[9],
                       int rx, int ry, int rz, double amp, uint64_t seed, double* out_pos,
                       int32_t* out_Z, double* out_lattice);

/* Kernel-level timing with CUDA events recorded on the handle's stream around
 * every launch.  gmd_profile(h, 1) clears and enables recording;
 * gmd_profile_read returns, per kernel name, the summed device time (ms) and
 * the number of launches.  names: NUL-separated, up to names_cap bytes;
 * total_ms / launches: arrays of at least *count entries (*count in = capacity). */
int gmd_profile(gmd_handle* h, int enable);
int gmd_profile_read(gmd_handle* h, char* names, int names_cap, double* total_ms, int* launches,
                     int* count);
/* process-wide number of kernel launches issued by this library so far */
int gmd_launch_count(int64_t* count);
/* the cudaStream_t every kernel of this handle is launched on */
int gmd_get_stream(gmd_handle* h, void** stream);

#ifdef __cplusplus
}
#endif
#endif /* GRAPHMD_B200_H */
