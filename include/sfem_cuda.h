/* sfem_cuda.h -- C-ABI of the B200-native spectral FEM Poisson solver.
 *
 * Drop-in boundary for the reference's hot path (algorithm (a), full
 * diagonalisation, and the standalone 1D expand/unexpand).  Plain pointers and
 * sizes only; every entry point returns 0 on success and a nonzero status
 * otherwise, with the message (the reference's sfem::Error text where one
 * exists) available from sfem_cuda_last_error() on the calling thread.
 * No C++ exception crosses this boundary (reference: types.hpp:9-18 throws
 * sfem::Error everywhere; include/sfem_b200.hpp rethrows it on the C++ side).
 *
 * Data layout ("dof layout"): an N-D grid function or coefficient tensor is
 * one dense FP64 array, row-major, last axis fastest, with per-axis extent
 * L_i = n_i*K_i - 1 in the interleaved dof order of the reference's dense
 * oracle (dof t = e*n + c: interior component c of element e; t = j*n - 1:
 * node j; reference proj/src/banded.cpp:9-15, oracle.cpp:64-144).  Device
 * tensors may pad the last axis to a pitch (in elements) >= L_{N-1}.
 * Coefficients of an axis are in the reference's frequency-major order
 * (grid1d.hpp:41-58).
 */
#ifndef SFEM_CUDA_H
#define SFEM_CUDA_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sfem_ctx_s* sfem_ctx;     /* device + stream                 */
typedef struct sfem_table_s* sfem_table; /* spectral table for one (n, K)   */
typedef struct sfem_plan_s* sfem_plan;   /* algorithm (a) solve plan        */

/* Library version (major*10000 + minor*100 + patch). */
int sfem_cuda_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* sfem_cuda_last_error(void);

/* Context on CUDA device `device` with its own stream.
 * Replaces the implicit process state of the reference (OpenMP pool,
 * FFTW plan cache: trig.cpp:27-67, poisson.cpp:81-87). */
int sfem_cuda_ctx_create(int device, sfem_ctx* out);
int sfem_cuda_ctx_destroy(sfem_ctx ctx);
/* The context's stream as a cudaStream_t (void*). */
int sfem_cuda_ctx_stream(sfem_ctx ctx, void** stream);

/* Spectral table for order n (1..9) and K >= 2 elements, built on the host
 * and uploaded.  Replaces TableSet::get / build_spectral_table
 * (reference poisson.hpp:54, spectral.hpp:316). */
int sfem_cuda_table_create(sfem_ctx ctx, int order, int elements, sfem_table* out);
int sfem_cuda_table_destroy(sfem_table table);
/* Host copies of the table's primaries (SpectralTable1D fields, spectral.hpp:281-312).
 * Any pointer may be NULL.  Sizes: values/norm_sq (K-1)*n; p (K-1)*n*(n-1);
 * interior_values n-1; interior_vectors (n-1)^2 row-major [i][l-1];
 * eig_coeff n*K-1 (eigenvalues_coeff_order, spectral.cpp:10-17). */
int sfem_cuda_table_export(sfem_table table, double* values, double* norm_sq, double* p,
                           double* interior_values, double* interior_vectors, double* eig_coeff);

/* Table files and the table cache (reference save_table / load_table /
 * build_and_save_table, spectral.hpp:316-330 / spectral.cpp:81-236, and
 * TableSet's cache directory, poisson.hpp:48-62 / poisson.cpp:49-73).
 *   SFEM_TABLE_TEXT    the reference's "SFEM1" text format (17 significant
 *                      digits), written byte for byte as save_table writes it
 *                      and read as load_table reads it (a cache directory the
 *                      reference filled is used as is);
 *   SFEM_TABLE_BINARY  "SFEMB1": the same primaries as raw doubles plus an
 *                      FNV-1a checksum (bit-exact, no text parse).
 * Loading sniffs the format, checks the header against (order, elements)
 * with load_table's messages, and rebuilds the derived data as the reference
 * does (spectral.cpp:209-235).  Writes go to a temporary name and are renamed
 * into place.
 *
 * sfem_cuda_ctx_set_table_cache: every later table of this context (table_create
 * and the plans' tables) is looked up as sfem_table_n<n>_K<K>.bin, then .txt
 * (the reference's name), under `dir`; an absent or stale entry is rebuilt and,
 * with SFEM_TABLE_CACHE_WRITE, written in the format SFEM_TABLE_CACHE_BINARY
 * selects (else text).  dir NULL or "" turns the cache off (the default).
 * sfem_cuda_table_file_build / _read work on the host only (no device) --
 * build_and_save_table, and load_table followed by the export of
 * sfem_cuda_table_export. */
enum { SFEM_TABLE_TEXT = 0, SFEM_TABLE_BINARY = 1 };
enum { SFEM_TABLE_CACHE_WRITE = 1, SFEM_TABLE_CACHE_BINARY = 2 };
int sfem_cuda_ctx_set_table_cache(sfem_ctx ctx, const char* dir, int flags);
int sfem_cuda_table_load(sfem_ctx ctx, const char* path, int order, int elements, sfem_table* out);
int sfem_cuda_table_save(sfem_table table, const char* path, int format);
int sfem_cuda_table_file_build(int order, int elements, const char* path, int format);
int sfem_cuda_table_file_read(const char* path, int order, int elements, double* values, double* norm_sq,
                              double* p, double* interior_values, double* interior_vectors, double* eig_coeff);

/* 1D line operations (reference eigenbasis.hpp:50-79):
 *   SFEM_OP_DECOMPOSE_WEIGHTED  lines::decompose_weighted  (FC_n, eigenbasis.cpp:63-101)
 *   SFEM_OP_DECOMPOSE           lines::decompose           (F_n,  eigenbasis.cpp:103-142)
 *   SFEM_OP_SYNTHESIZE          lines::synthesize          (F_n^-1, eigenbasis.cpp:144-225)
 * on `count` lines of length L = n*K-1, line b at in + b*in_pitch (dof layout
 * for the analyses, coefficient layout for synthesis).  In-place allowed when
 * in == out and the pitches agree. */
enum { SFEM_OP_DECOMPOSE_WEIGHTED = 0, SFEM_OP_DECOMPOSE = 1, SFEM_OP_SYNTHESIZE = 2 };
/* Element stencils on the same dof-layout lines (grid1d.cpp:7-47):
 *   SFEM_OP_APPLY_MASS       apply_mass_1d       y = M v
 *   SFEM_OP_APPLY_STIFFNESS  apply_stiffness_1d  y = A v
 * with the reference-element matrices of the table's order (no h scaling, as
 * the reference).  Boundary nodes are absent from the dof layout.  Together
 * with SFEM_OP_DECOMPOSE_WEIGHTED, APPLY_MASS gives decompose's
 * DirectRoute::MassApply (eigenbasis.cpp:469-470). */
enum { SFEM_OP_APPLY_MASS = 3, SFEM_OP_APPLY_STIFFNESS = 4 };
int sfem_cuda_lines_device(sfem_table table, int op, long long count, const double* d_in,
                           long long in_pitch, double* d_out, long long out_pitch, void* stream);
/* The same three transforms on lines with an element stride: position t of
 * line b at d_in[t*pos_stride + b*line_stride] (and the same offsets in
 * d_out; in place when d_in == d_out).  pos_stride = count, line_stride = 1 is
 * the slot-major tile of the reference's batched kernels ("the value at
 * position j of line b sits at [j*count + b]", eigenbasis.hpp:66-69) in the
 * dof / coefficient layout; pos_stride = 1 is sfem_cuda_lines_device. */
int sfem_cuda_lines_strided_device(sfem_table table, int op, long long count, const double* d_in, double* d_out,
                                   long long pos_stride, long long line_stride, void* stream);
/* lines::decompose_weighted_block / synthesize_block (eigenbasis.hpp:70-73,
 * eigenbasis.cpp:248-444) with the reference's own arguments: slot-major
 * class tiles, nodal (K+1) x count (boundary slots included; ignored by the
 * analyses, written as 0 by the synthesis), interior K*(n-1) x count
 * element-major (NULL for n = 1), coeffs (n*K-1) x count frequency-major,
 * all addressed [j*count + b].  SFEM_OP_DECOMPOSE_WEIGHTED / _DECOMPOSE read
 * the class tiles and write coeffs; SFEM_OP_SYNTHESIZE reads coeffs and
 * writes the class tiles.  Any count >= 1 (the reference uses <= 32,
 * poisson.cpp:231). */
int sfem_cuda_lines_block_device(sfem_table table, int op, long long count, double* d_nodal, double* d_interior,
                                 double* d_coeffs, void* stream);
/* Same on host buffers (dense, pitch = L); host<->device copies included. */
int sfem_cuda_lines_host(sfem_table table, int op, long long count, const double* h_in, double* h_out);
/* materialize_eigenvector (spectral.hpp:330, spectral.cpp:238-265): the grid
 * values of eigenvector (k, l) (k = 0: l = 1..n-1; k >= 1: l = 1..n) in the
 * dof layout (n*K-1 doubles, host memory), from the table's primaries. */
int sfem_cuda_table_eigenvector(sfem_table table, int k, int l, double* out);

/* Solve plan for  -sum_i a_i d^2u/dx_i^2 + shift*u = f  on the box
 * prod [0, lengths_i] with homogeneous Dirichlet data, orders n_i and K_i
 * elements per axis (reference ProblemSpec, poisson.hpp:29-41; a_i = 1 there).
 * `coefficients` may be NULL (all ones).  Validation and the nonpositive-
 * symbol check follow ProblemSpec::validate (poisson.cpp:32-47) and
 * detail::scale_by_symbol (poisson.cpp:573-631), with their messages.
 * dim 1..4. */
int sfem_cuda_plan_create(sfem_ctx ctx, int dim, const int* orders, const int* elements,
                          const double* lengths, const double* coefficients, double shift, sfem_plan* out);
int sfem_cuda_plan_destroy(sfem_plan plan);
/* Extents L_i (dim entries), default device pitch of the last axis, total unknowns. */
int sfem_cuda_plan_shape(sfem_plan plan, long long* extents, long long* pitch, long long* unknowns);
/* Kernel launches per solve (2N-1 for the fused schedule). */
int sfem_cuda_plan_launches(sfem_plan plan, int* launches);

/* Algorithm of the plan's solves (reference SolveOptions::algorithm,
 * poisson.hpp:64-70): 0 = FullDiagonalization (default), 1 =
 * PartialDiagonalization (poisson.cpp:671-745: expansions along axes 1..N-1,
 * a banded SPD solve along axis 0 per frequency line; dimension >= 2).  An
 * indefinite line raises the reference's error in the synchronous host
 * entry points. */
int sfem_cuda_plan_set_algorithm(sfem_plan plan, int algorithm);

/* Device-resident solve, in place: d_data holds the load (dof layout, last
 * axis padded to `pitch` elements) and receives u.  Replaces
 * solve_with_load's timed core run_full_diagonalization (poisson.cpp:637-669,
 * timed region 781-785).  stream NULL = the context stream.  Any pitch >=
 * L_{N-1} may be passed per call (the plan's own buffers keep their size).
 * Plan-owned scratch is shared by all of the plan's solves: a solve issued on
 * a different stream than the previous one is ordered after it (event wait),
 * so one plan never runs two solves concurrently; use one plan per stream for
 * concurrent solves.  The same holds for a context's global FFT scratch
 * across its plans and line calls. */
int sfem_cuda_solve_device(sfem_plan plan, double* d_data, long long pitch, void* stream);

/* Host solve: dense dof-layout load in, dense u out (h_u may equal h_load).
 * Host->device and device->host copies are inside.  `seconds` (may be NULL)
 * receives the device-timed solve alone (SolveReport::seconds_solve). */
int sfem_cuda_solve_host(sfem_plan plan, const double* h_load, double* h_u, double* seconds);

/* Pipelined host solves of `count` independent loads with this plan (e.g.
 * several right-hand sides): the host->device copy of problem i+1 and the
 * device->host copy of i-1 run while i is solved (three device slots, three
 * streams).
 * Pinned host buffers are needed for the copies to overlap. */
int sfem_cuda_solve_host_batch(sfem_plan plan, long long count, const double* const* h_loads, double* const* h_us);

/* Host solve in the reference's GridFunctionND layout (ndgrid.hpp:43-57): 2^dim
 * class arrays, mask bit i set = element-interior indexing on axis i, class
 * extents K_i+1 (nodal, boundary slots included) or K_i*(n_i-1); row-major.
 * Boundary slots of the result are zero (enforce_boundary, ndgrid.cpp:34-45). */
int sfem_cuda_solve_classes(sfem_plan plan, const double* const* h_load_classes, double* const* h_u_classes,
                            double* seconds);

/* Timing helper for benchmarks: `reps` solves of d_data back to back on the
 * plan stream, bracketed by CUDA events; per-sweep-kernel times (ms, averaged
 * over reps) into kernel_ms[0 .. launches-1] when non-NULL. */
int sfem_cuda_solve_device_timed(sfem_plan plan, double* d_data, long long pitch, int reps, double* total_ms,
                                 double* kernel_ms);

/* ---- The steps either side of the solve, on the device ----
 * Built-in right-hand sides (the reference's ScalarField callbacks cannot
 * cross to the device; these are its manufactured cases, cases.cpp:11-55,
 * plus the product of sines of BASELINE config 3):
 *   SFEM_FIELD_CONSTANT   f = params[0]                       (cases "constantNd": 1)
 *   SFEM_FIELD_SINES      f = params[0] * prod_i sin(params[1+i] * pi * x_i);
 *                         exact u = f / (sum_i a_i (params[1+i] pi)^2 + shift)
 *   SFEM_FIELD_SIN1D / _POISSON2D / _POISSON3D
 *                         f = -Lap u + shift u for the reference's u (unit
 *                         coefficients only, as make_problem, cases.cpp:81-95) */
enum {
  SFEM_FIELD_CONSTANT = 0, SFEM_FIELD_SINES = 1, SFEM_FIELD_SIN1D = 2, SFEM_FIELD_POISSON2D = 3,
  SFEM_FIELD_POISSON3D = 4
};
/* FEM load of a field on the plan's box into d_load (dof layout, pitch):
 * replaces fem_load_average (poisson.cpp:471-569; (n+1)-point Gauss rule per
 * axis, boundary contributions dropped).  Deterministic (no atomics). */
int sfem_cuda_fem_load(sfem_plan plan, int field, const double* params, int nparams, double* d_load,
                       long long pitch, void* stream);
/* d_y = A d_v, A the plan's FEM operator sum_i f_i (x)_{j!=i} M_j (x) S_i +
 * shift (x) M_j; replaces apply_operator (poisson.cpp:749-769).  v != y. */
int sfem_cuda_apply_operator(sfem_plan plan, const double* d_v, double* d_y, long long pitch, void* stream);
/* residual_rel = max|A u - f| / max|f| (1 if f == 0 everywhere) on the device,
 * as SolveReport::residual_rel (poisson.cpp:785-789).  Synchronous. */
int sfem_cuda_residual(sfem_plan plan, const double* d_u, const double* d_f, long long pitch, double* residual_rel);
/* error = max over the dofs of |u - u_exact| for a field with a known solution
 * (SINES and the cases); replaces max_error_vs (ndgrid.cpp:80-101; boundary
 * slots, where u = 0 = u_exact, are not stored).  Synchronous. */
int sfem_cuda_max_error(sfem_plan plan, int field, const double* params, int nparams, const double* d_u,
                        long long pitch, double* error);

/* The reference's end-to-end solve(spec, options) (poisson.cpp:796-808) of a
 * built-in field, every step on the device: FEM load, solve, optionally the
 * residual check, and the uniform error for fields with a known solution.
 * report[4] = {seconds_load, seconds_solve, residual_rel (NaN unless
 * compute_residual), error_uniform (NaN for CONSTANT)}; h_u (dense dof
 * layout, may be NULL) receives the solution. */
int sfem_cuda_solve_field(sfem_plan plan, int field, const double* params, int nparams, int compute_residual,
                          double* h_u, double* report);
/* apply_operator (poisson.cpp:749-769) on dense host dof tensors. */
int sfem_cuda_apply_operator_host(sfem_plan plan, const double* h_v, double* h_y);

/* ---- Multi-GPU slab decomposition (one process / context per GPU) ----
 * Rank r owns the x-slab of axis-0 dof rows [x0, x0+lx) of the global dof
 * tensor (all other axes; last axis padded to xpitch) and, between the two
 * all-to-all exchanges, the y-slab of axis-1 rows [y0, y0+ly) stored as
 * [ly][R][ypitch] with axis 0 contiguous (R = prod of the extents of axes
 * 2..N-1).  One solve = FORWARD_LOCAL(x), PACK1(x->buf), all-to-all(buf),
 * UNPACK1(buf->y), AXIS0(y), PACK2(y->buf), all-to-all(buf, reverse counts),
 * UNPACK2(buf->x), INVERSE_LOCAL(x).  The exchanges are the caller's (NCCL,
 * e.g. torch.distributed.all_to_all_single); split sizes from dist_shape.
 * Replaces the same run_full_diagonalization (poisson.cpp:637-669), sharded. */
typedef struct sfem_dist_s* sfem_dist;
enum {
  SFEM_DIST_FORWARD_LOCAL = 0, SFEM_DIST_PACK1 = 1, SFEM_DIST_UNPACK1 = 2, SFEM_DIST_AXIS0 = 3,
  SFEM_DIST_PACK2 = 4, SFEM_DIST_UNPACK2 = 5, SFEM_DIST_INVERSE_LOCAL = 6
};
int sfem_cuda_dist_create(sfem_ctx ctx, int dim, const int* orders, const int* elements, const double* lengths,
                          const double* coefficients, double shift, int nranks, int rank, sfem_dist* out);
int sfem_cuda_dist_destroy(sfem_dist dist);
/* info[10] = {x0, lx, y0, ly, x-slab elements, y-slab elements, exchange
 * buffer elements, xpitch, ypitch, R}; send/recv_counts[nranks] (elements) of
 * exchange 1 (exchange 2 swaps them); either may be NULL. */
int sfem_cuda_dist_shape(sfem_dist dist, long long* info, long long* send_counts, long long* recv_counts);
int sfem_cuda_dist_phase(sfem_dist dist, int phase, double* d_x, double* d_y, double* d_buf, void* stream);

/* ---- The same slab solve with the library owning the exchange (NCCL) ----
 * A C or C++ host needs no collective of its own: the plan creates an NCCL
 * communicator from a unique id (made on one rank by sfem_cuda_nccl_unique_id
 * and handed to the others by whatever the host uses: MPI, a socket, a file),
 * allocates the exchange buffers and the y-slab, and one call runs the whole
 * solve on this rank's x-slab d_x ([lx][L1]..[L_{N-1}], last axis padded to
 * xpitch; in place).  Both all-to-all exchanges are grouped ncclSend/ncclRecv
 * on a second stream, split into `chunks` pieces (0 = default 4; fewer if the
 * in-place axis-0 sweep would need more than 32 row segments) so that chunk c
 * travels over NVLink while chunk c+1 is swept: exchange 1 behind the forward
 * sweeps of x-row chunks, exchange 2 behind the fused axis-0 sweeps of y-row
 * chunks.  libnccl.so.2 is opened at run time (dlopen), not linked.
 * Replaces run_full_diagonalization (poisson.cpp:637-669), sharded. */
#define SFEM_NCCL_UNIQUE_ID_BYTES 128
int sfem_cuda_nccl_unique_id(void* id /* SFEM_NCCL_UNIQUE_ID_BYTES */);
int sfem_cuda_dist_comm_init(sfem_dist dist, const void* id, int chunks);
int sfem_cuda_dist_solve(sfem_dist dist, double* d_x, void* stream);
/* After a solve: phase_ms[6] = {forward local + pack, exchange 1 left exposed,
 * axis 0, exchange 2 left exposed, unpack + inverse local, whole solve} from
 * CUDA events (synchronises on the last one) and the bytes this rank sent to
 * other ranks per solve.  Either pointer may be NULL. */
int sfem_cuda_dist_solve_stats(sfem_dist dist, double* phase_ms, long long* bytes_sent);
/* Chunk schedule and buffers without a communicator, and all `n` ranks of a
 * solve run in one process on one device with the messages moved by device
 * copies (the single-GPU check of the chunked schedule: same phases, chunks and
 * message lists as sfem_cuda_dist_solve). */
int sfem_cuda_dist_setup(sfem_dist dist, int chunks);
/* The messages of exchange `step` (1 or 2), chunk `chunk`, of this rank, in
 * issue order: n_send sends then n_recv receives, each (peer, offset, count) in
 * doubles (offsets into the send / receive exchange buffer).  peers / offsets /
 * counts (capacity entries each) may be NULL to query the counts. */
int sfem_cuda_dist_messages(sfem_dist dist, int step, int chunk, int capacity, int* n_send, int* n_recv, int* peers,
                            long long* offsets, long long* counts);
int sfem_cuda_dist_solve_group(sfem_dist* dists, int n, double* const* d_xs, void* stream);

/* ---- Multi-GPU with the exchanges fused into the sweeps over NVLink ----
 * 3-D problems whose axes 0 and 1 have K = 64 tables (config 4), 1..8 ranks,
 * one process per GPU.  No NCCL on the data path: the axis-1 forward sweep
 * TMA-stores each finished tile straight into the owning rank's y-slab (peer
 * memory), and the fused axis-0 sweep (forward + divide + inverse) stores its
 * tiles straight back into the source ranks' x-slabs.  Rank r's buffers are
 * plan-owned: x-slab [lx][L1][pitch] (axis-0 rows x0.., laid out x, y, z) and
 * y-slab [ly][L0][pitch] (axis-1 rows y0..).  One solve:
 *   PEER_FORWARD, PEER_BARRIER, PEER_AXIS0, PEER_BARRIER, PEER_INVERSE.
 * Replaces run_full_diagonalization (poisson.cpp:637-669), sharded. */
typedef struct sfem_peer_s* sfem_peer;
enum { SFEM_PEER_FORWARD = 0, SFEM_PEER_AXIS0 = 1, SFEM_PEER_INVERSE = 2, SFEM_PEER_BARRIER = 3 };
int sfem_cuda_peer_create(sfem_ctx ctx, int dim, const int* orders, const int* elements, const double* lengths,
                          const double* coefficients, double shift, int nranks, int rank, sfem_peer* out);
int sfem_cuda_peer_destroy(sfem_peer peer);
/* info[8] = {x0, lx, y0, ly, x-slab elements, y-slab elements, pitch, nranks} */
int sfem_cuda_peer_shape(sfem_peer peer, long long* info);
/* This rank's plan-owned device buffers (x-slab, y-slab, barrier flag words). */
int sfem_cuda_peer_buffers(sfem_peer peer, void** x_slab, void** y_slab, void** flags);
/* Every rank's buffers as mapped in this process (own slot = own buffers;
 * others from sfem_cuda_ipc_open_handle).  flags NULL: no device barrier
 * (all ranks on one device, phases run rank after rank: the loopback check). */
int sfem_cuda_peer_bind(sfem_peer peer, void* const* x_slabs, void* const* y_slabs, void* const* flags);
int sfem_cuda_peer_phase(sfem_peer peer, int phase, void* stream);
/* After synchronising `stream` (NULL = context stream): the epoch of a device
 * barrier that gave up after 20 s because a peer never arrived (0 = none).
 * A barrier that times out returns instead of trapping, so the context stays
 * usable and every rank can agree on a fallback. */
int sfem_cuda_peer_status(sfem_peer peer, void* stream, long long* timed_out_epoch);
/* CUDA IPC of a device allocation between the ranks' processes (64-byte handles). */
int sfem_cuda_ipc_get_handle(void* d_ptr, void* handle);
int sfem_cuda_ipc_open_handle(const void* handle, void** d_ptr);
int sfem_cuda_ipc_close(void* d_ptr);

#ifdef __cplusplus
}
#endif
#endif
