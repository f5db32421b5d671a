/*
 * fieldtess_cuda.h -- C-ABI of the B200 (sm_100a) layered-field engine.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `fieldtess` (arXiv 1804.09152).  The reference has no native code: its
 * compute layer is a set of numba kernels that take raw numpy arrays and
 * write into caller-preallocated outputs, signalling errors through flag
 * arrays (`fieldtess/_kernels.py`).  Each entry point below replaces one
 * stage of that pipeline (citations are `path:line` under the reference's
 * `pkg/src/fieldtess/`).
 *
 * Conventions
 *   - `extern "C"`, plain pointers and sizes, no exceptions cross the ABI.
 *   - Canonical matrices are CSC exactly as the reference stores them
 *     (`sparse.py:27-57`): int32 `col_ptr[n_cols+1]`, int32 `row_idx[cap]`,
 *     values `double` (FT_F64) or `float` (FT_F32).  The layered field PHI is
 *     (n_cells+1) x n_vertices: column = vertex, row 0 = base layer,
 *     row r = cell r-1 (`field.py:95-130`).
 *   - Between Euler steps the engine keeps PHI in a hybrid layout
 *     (ft_tiled): a column with at most two entries lives in four dense
 *     per-column arrays (row signature, second row, first value, second
 *     value); a wider column lives in an overflow pool.  A kernel reads a
 *     neighbour's entries with no descriptor indirection and writes its own
 *     column at a fixed address, so the step has no inter-CTA dependency
 *     and no placement scan; canonical CSC is produced by ft_compact at the
 *     API boundary.
 *   - The Laplacian is passed as `lap.mat_t` (L^T in CSC), which is
 *     byte-identical to L in CSR with ascending neighbour index including
 *     the diagonal (`mesh.py:379-431`).
 *   - Every pointer argument except the host-side `ft_params*` and the
 *     descriptor structs themselves is DEVICE memory owned by the caller.
 *     Calls only enqueue work on `stream` (a `cudaStream_t`, passed as
 *     void*); results are read back by the caller.
 *   - Return value: FT_OK or an FT_ERR_* code; `ft_last_error()` returns a
 *     thread-local message for the last failure.
 */
#ifndef FIELDTESS_CUDA_H
#define FIELDTESS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FT_ABI_VERSION 6

/* return codes (mapped onto the reference's TessError subclasses,
 * `errors.py:9-75`, by the Python host layer) */
#define FT_OK              0
#define FT_ERR_SHAPE       1  /* ShapeError                                  */
#define FT_ERR_NUMERICAL   2  /* NumericalBlowupError(column, step)          */
#define FT_ERR_CAPACITY    3  /* output capacity too small: grow, retry
                                 (ensure_capacity, sparse.py:212-232)        */
#define FT_ERR_CUDA        4  /* CUDA runtime failure                        */
#define FT_ERR_PATTERN     5  /* PatternViolationError (sparse.py:389-394)   */
#define FT_ERR_ARG         6  /* bad argument (null pointer, bad dtype, ...)  */

/* value dtypes */
#define FT_F64 0   /* EXACT mode: bitwise identical to the reference       */
#define FT_F32 1   /* FAST mode: fp32 storage, fp64 in-register arithmetic  */

/* Laplacian flags */
#define FT_LAP_EXPLICIT 0  /* use the stored values                           */
#define FT_LAP_UNIFORM  1  /* values are exactly 1.0/deg(j) off-diagonal and
                              -1.0 on the diagonal (mesh.py:392-400): they are
                              recomputed in registers and never read          */
#define FT_LAP_PACKED   2  /* with FT_LAP_UNIFORM: lap_t->values points to the
                              packed neighbour table of ft_laplacian_pack (the
                              uniform values are never read, so the slot
                              carries the table); col_ptr / row_idx stay valid */
#define FT_LAP_CHECK_FINITE 4  /* tiled input of unknown origin: check its
                              values for NaN / Inf (automatic for canonical
                              input and after any non-finite output)        */
#define FT_LAP_SYMMETRIC 8 /* the pattern of L^T is symmetric (column j is read
                              by exactly the columns it reads; every mesh
                              Laplacian of mesh.py:379-431): enables
                              active-set stepping -- a column whose closed
                              one-ring did not change in the previous step is
                              not recomputed (its value is already in place)  */
#define FT_HINT_DENSE_BAND 16 /* performance hint only (results are identical
                              with or without it): the field's band is dense
                              -- many columns with three layer rows in their
                              one-ring (reference configs[4], 65,536 seeds on
                              10M vertices) -- so the three-row kernel trades
                              registers for occupancy.  The Python layer sets
                              it when nnz - n_cols >= 2^21; it also enables
                              the four-row kernel                            */
#define FT_HINT_FOUR_ROW 32 /* performance hint only: launch the four-row
                              kernel (a no-op unless the three-row kernel
                              leaves >= 48K columns, but a launch per step).
                              The Python layer sets it for young fields
                              (nnz - n_cols < n_cols / 16: a band still
                              forming from init_field), where those columns
                              are many in the first steps                    */

/* status codes written into ft_step_stats.status / evolve control[1] */
#define FT_STATUS_OK           0
#define FT_STATUS_NAN          1   /* NumericalBlowupError                    */
#define FT_STATUS_PATTERN      2   /* PatternViolationError                   */
#define FT_STATUS_OVERFLOW     3   /* tiled work buffer too small             */
#define FT_STATUS_CONVERGED    4
#define FT_STATUS_MAXSTEPS     5
#define FT_STATUS_OUT_OVERFLOW 6   /* canonical output too small: grow it and
                                      call ft_compact                         */
#define FT_STATUS_HALO_OVERFLOW 7  /* partitioned field: a halo column holds
                                      more entries than the exchange slots    */

/* CouplingParams (field.py:34-71).  Host memory. */
typedef struct {
    double w, a, e, e_base, mu, dt;
} ft_params;

/* Canonical CSC.  `values` dtype given by the call's dtype argument. */
typedef struct {
    int32_t  n_rows;
    int32_t  n_cols;
    int32_t* col_ptr;     /* [n_cols+1]                                   */
    int32_t* row_idx;     /* [capacity]                                   */
    void*    values;      /* [capacity] double or float                   */
    int64_t  capacity;
} ft_csc;

/* Hybrid working layout of a field (see Conventions).  Column j:
 *   sig[j] == -1            no entry
 *   0 <= sig[j] < 2^30      one entry: row sig[j], value v0[j]
 *   sig[j] >= 2^30          two entries: rows sig[j] - 2^30 < aux[j],
 *                           values v0[j], v1[j]
 *   sig[j] <= -3            -sig[j] entries at pool_idx / pool_val
 *                           [aux[j], aux[j] - sig[j])
 * The dense arrays have n_cols entries; pool offsets index pool_idx /
 * pool_val.  A view of a column range offsets the four dense pointers.
 * At most 2^30 layer rows (FT_ERR_SHAPE otherwise). */
typedef struct {
    int32_t  n_rows;
    int32_t  n_cols;
    int32_t* sig;         /* [n_cols] row signature (see above)            */
    int32_t* aux;         /* [n_cols] second row / pool offset             */
    void*    v0;          /* [n_cols] first value (double or float)        */
    void*    v1;          /* [n_cols] second value                         */
    int32_t* pool_idx;    /* [capacity] rows of the pool columns           */
    void*    pool_val;    /* [capacity] values of the pool columns         */
    int64_t  capacity;    /* pool entries                                  */
} ft_tiled;

#define FT_SIG_PAIR  (1 << 30)
#define FT_SIG_EMPTY (-1)

/* One step's statistics, device resident.  Mirrors StepStats
 * (field.py:74-92) plus the error flags the reference signals through
 * `nan_col` / `bad_col` arrays (_kernels.py:165-176, 231-233). */
typedef struct {
    double  max_delta;        /* max_j max_p |v' - phi_old|  (field.py:271)  */
    double  base_mass;        /* sum_j base mass             (field.py:270)  */
    int64_t nnz_phi;          /* nnz of the output field                     */
    int64_t nnz_skel;         /* interest-skeleton nnz of the step           */
    int32_t status;           /* FT_STATUS_*                                 */
    int32_t nan_col;          /* first column that produced NaN, or -1       */
    int32_t bad_col;          /* first column with a pattern violation, -1   */
    int32_t bad_row;          /* offending row in `bad_col`                  */
    int32_t bad_is_lt;        /* 0: violation in PHI, 1: in Lt               */
    int32_t step;             /* 1-based step index within the call         */
    int64_t needed;           /* capacity needed when status is an overflow  */
} ft_step_stats;

/* -- library ------------------------------------------------------------- */
int         ft_abi_version(void);
const char* ft_last_error(void);

/* Scratch `workspace` for a field of n_vertices columns (device control
 * block with the running statistics, the active list, the column lists of
 * the wide kernels, per-column skeleton sizes and activity stamps,
 * compaction scan space; 17 bytes per column).  Zero it once with
 * ft_workspace_init; then reuse it for every call on fields of that size.
 * It carries the active-set state between the steps of one field. */
size_t ft_workspace_bytes(int32_t n_vertices);
int    ft_workspace_init(void* workspace, size_t bytes, void* stream);

/* Canonical CSC -> hybrid layout (columns with more than two entries take
 * pool space with one atomic per warp).  A non-finite value raises the
 * workspace's sticky non-finite flag, so the next step checks its inputs.
 * stats->status = FT_STATUS_OVERFLOW and stats->needed when the pool is
 * too small. */
int ft_tiled_from_csc(const ft_csc* src, ft_tiled* dst, int32_t dtype, void* workspace,
                      size_t ws_bytes, ft_step_stats* stats, void* stream);

/* Packed neighbour table of L^T for the tier-1 kernel: int16[n_cols][8],
 * column j's entries as deltas u - (col_base + j) in stored order (the
 * reference accumulation order), unused slots -32768.  A column with more
 * than 8 entries or a delta outside int16 gets all slots -32768 and is read
 * from col_ptr / row_idx (counted in *n_csr, device int32).  One coalesced
 * 16-byte load per column replaces the col_ptr -> row_idx dependency chain.
 * `pack` must be 16-byte aligned. */
int ft_laplacian_pack(const ft_csc* lap_t, int32_t col_base, int16_t* pack, int32_t* n_csr,
                      void* stream);

/* -- the fused Euler step ------------------------------------------------ */
/* One explicit Euler step, canonical in -> canonical out.  Replaces the
 * whole pipeline of field.step (field.py:198-286):
 *   sparse.spgemm (sparse.py:279-330; _kernels.py:14-74)      Lt = PHI L^T
 *   sparse.build_skeleton (sparse.py:345-371; _kernels.py:96-150)
 *   sparse.expand_to_skeleton x2 (sparse.py:374-396; _kernels.py:153-176)
 *   _kernels.update_kernel (_kernels.py:179-238)
 *   _kernels.column_sums_counts + normalize_compact (_kernels.py:241-282)
 * as: ft_tiled_from_csc(phi_in -> scratch_in), the fused step kernels
 * (scratch_in -> scratch_out), then ft_compact into `phi_out`.  `stats`
 * (device, one record) receives the statistics; on FT_STATUS_OVERFLOW
 * (scratch pools) / FT_STATUS_OUT_OVERFLOW (phi_out) stats->needed holds
 * the required capacity and the input is intact. */
int ft_step(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
            ft_tiled* scratch_in, ft_tiled* scratch_out, ft_csc* phi_out, int32_t dtype,
            const ft_params* params, void* workspace, size_t ws_bytes,
            ft_step_stats* stats, void* stream);

/* ft_step with its device time split at the kernel-group boundaries into
 * phase_ms[5] (host, milliseconds; synchronises the stream), reported in
 * the reference's five StepStats phase slots (field.py:220-285):
 *   [0] skeleton_time   layout conversion + active-column selection (prep)
 *   [1] spgemm_time     band kernel: fused L^T gather + update + normalise
 *                       of the one/two-layer columns
 *   [2] expand_time     three-layer kernel
 *   [3] update_time     warp / serial kernels of the wider columns
 *   [4] normalize_time  statistics finalize + compaction to CSC */
int ft_step_phases(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
                   ft_tiled* scratch_in, ft_tiled* scratch_out, ft_csc* phi_out,
                   int32_t dtype, const ft_params* params, void* workspace,
                   size_t ws_bytes, ft_step_stats* stats, float* phase_ms, void* stream);

/* One step from a hybrid-layout input, for callers that drive the step
 * sequence themselves (bench.py brackets the column kernels with CUDA
 * events).  `out_id` (0 / 1) names the target buffer: a sequence of steps
 * ping-pongs between two buffers with ids 0 and 1 (ft_evolve: work_a = 0,
 * work_b = 1), starting after ft_tiled_from_csc into buffer 1.
 *   FT_PHASE_COLUMNS   the column kernels: active list, band kernel (one
 *                      lane per column: closed form / two-row update), the
 *                      three- and four-row lane kernels and the
 *                      warp-cooperative kernel for wide columns;
 *   FT_PHASE_FINALIZE  the serial pass over the columns beyond the warp
 *                      kernel's staging capacity (rare), the statistics
 *                      record into `stats` (device), the next step's mode.
 * Both phases take the same arguments (the finalize pass reads the step's). 
 * ft_evolve issues exactly this sequence. */
#define FT_PHASE_COLUMNS  1
#define FT_PHASE_FINALIZE 2
int ft_step_run(const ft_csc* lap_t, int32_t lap_flags, const ft_tiled* in,
                ft_tiled* out, int32_t out_id, int32_t dtype, const ft_params* params,
                void* workspace, size_t ws_bytes, int32_t phases,
                ft_step_stats* stats, void* stream);

/* Tiled -> canonical CSC (device-wide scan of column counts, then a
 * coalesced copy).  stats->nnz_phi / needed / status report the result
 * (FT_STATUS_OUT_OVERFLOW when dst is too small). */
int ft_compact(const ft_tiled* src, ft_csc* dst, int32_t dtype, void* workspace,
               size_t ws_bytes, ft_step_stats* stats, void* stream);

/* Up to `max_steps` steps from the canonical `phi_in` (converted into
 * work_b), ping-ponging between the hybrid buffers a (odd steps) and b
 * (even steps), stopping on the
 * device as soon as a step converges (max_delta < tol and base_mass <
 * base_threshold; field.py:316-317) or fails (NaN / pattern violation /
 * tiled overflow).  The last good field is then compacted into `phi_out`.
 * Replaces the loop of field.evolve (field.py:289-321).
 * `trace` (device, max_steps records) receives one ft_step_stats per
 * executed step (plus the failing one); `control` (device, 4 x int64)
 * receives {steps_done, status, needed_capacity, compacted(0/1)}. */
int ft_evolve(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
              ft_tiled* work_a, ft_tiled* work_b, ft_csc* phi_out,
              int32_t dtype, const ft_params* params, int32_t max_steps,
              double tol, double base_threshold, void* workspace,
              size_t ws_bytes, ft_step_stats* trace, int64_t* control,
              void* stream);

/* -- partitioned fields (one rank per GPU) ------------------------------- */
/* A field of n_vertices columns split into contiguous owned column ranges,
 * one per rank.  Every rank keeps two tiled buffers over its LOCAL columns:
 * the sorted union of its owned columns and its halo (the non-owned columns
 * its owned L^T columns read), numbered 0 .. n_local-1 in global order, so
 * the owned ones form the range [col_begin, col_begin + col_count).  One
 * Euler step is
 *   ft_domain_step     owned columns -> out (entries [0, step_capacity))
 *   ft_halo_pack       per peer: the owned columns the peer reads -> message
 *   (all-gather of the per-rank records; ncclAllGather)
 *   ft_domain_combine  global statistics + the evolve stop test, identical
 *                      on every rank (fixed rank order)
 *   (message exchange with the peers; ncclSend / ncclRecv)
 *   ft_halo_unpack     per peer: message -> halo columns of out (entries
 *                      from step_capacity on, `slots` per column); a halo
 *                      column that changed stamps its owned readers active
 * With FT_LAP_SYMMETRIC a rank steps its active set only (as ft_evolve);
 * ranks decide full / active steps independently.  Every launch is a
 * device-side no-op once the control block's done flag is set (converged /
 * max steps / failure), so a host loop may enqueue steps ahead and read
 * ft_domain_control only every few steps.  The owned columns are bitwise
 * identical to the single-GPU ft_evolve.  Host reference:
 * paper_1804_09152_b200/distributed.py (the reference is single-process). */
typedef struct {
    int32_t col_begin;       /* first owned local column                    */
    int32_t col_count;       /* number of owned columns                     */
    int64_t step_capacity;   /* entries the step may use in `out`          */
    const int32_t* report_ids;  /* nullable, device [col_count]: the caller's
                                   vertex ids of the owned columns; NaN /
                                   pattern errors report them              */
    int32_t out_id;          /* 0 / 1: which of the two buffers `out` is   */
    int32_t pad;
} ft_domain;

#define FT_HALO_FORCE 1      /* pack / unpack even when done is set         */

/* One step of the owned columns (all kernels) plus the local statistics
 * record.  lap_rows: the owned columns of L^T (n_rows = n_local, n_cols =
 * col_count, local row indices).  workspace: ft_workspace_bytes(n_local).
 * `record` (device) receives the local ft_step_stats. */
int ft_domain_step(const ft_csc* lap_rows, int32_t lap_flags, const ft_tiled* in,
                   ft_tiled* out, int32_t dtype, const ft_params* params,
                   const ft_domain* dom, void* workspace, size_t ws_bytes,
                   ft_step_stats* record, void* stream);

/* Size of a halo message for n columns: int32 counts[n], then int32
 * rows[n*slots], then values[n*slots] (dtype). */
int64_t ft_halo_bytes(int32_t n_cols, int32_t slots, int32_t dtype);

/* Pack columns cols[0..n) (device int32) of `src` into `msg`.  Skipped when
 * done is set or record->status is not OK (unless FT_HALO_FORCE).  A column
 * with more than `slots` entries turns record->status into
 * FT_STATUS_HALO_OVERFLOW and raises *need (device int32) to its count. */
int ft_halo_pack(const ft_tiled* src, const int32_t* cols, int32_t n, int32_t slots,
                 int32_t dtype, void* msg, ft_step_stats* record, int32_t* need,
                 void* workspace, int32_t flags, void* stream);

/* Column cols[i] of `dst` <- message entry i: in the dense arrays when it
 * holds at most two entries, else at pool entries [region + i*slots,
 * region + i*slots + count).  With `prev` (the step's input buffer) and the
 * readers CSR (readers_ptr[n+1], readers_idx: the owned local columns that
 * read cols[i]), a column that differs from its copy in `prev` stamps its
 * readers active for the next step.  Skipped when done is set (unless
 * FT_HALO_FORCE). */
int ft_halo_unpack(ft_tiled* dst, const int32_t* cols, int32_t n, int32_t slots,
                   int32_t dtype, const void* msg, int64_t region, void* workspace,
                   int32_t flags, const ft_tiled* prev, const int32_t* readers_ptr,
                   const int32_t* readers_idx, void* stream);

/* Global record from the all-gathered per-rank records (device, `world`
 * records in rank order): max of max_delta, base_mass summed in rank
 * order, nnz sums; the failure of highest priority (pattern > NaN >
 * overflow > halo overflow), reported at its lowest column over the ranks.  Applies the stop test of ft_evolve
 * (field.py:316-317) and writes trace[steps_done]; `needed` is the local
 * rank's. */
int ft_domain_combine(const ft_step_stats* records, int32_t world, int32_t rank,
                      int32_t max_steps, double tol, double base_threshold,
                      void* workspace, ft_step_stats* trace, void* stream);

/* Control block: out (device int64[3]) <- {steps_done, status, needed};
 * with set_steps >= 0 first resets it to steps_done = set_steps, not done,
 * status OK (rewind after a capacity failure). */
int ft_domain_control(void* workspace, int32_t set_steps, int64_t* out, void* stream);

/* -- mesh generation, geometry, uniform Laplacian (mesh.py:20-246, 379-431) */
/* Device replacements of the host generators, bitwise equal to the
 * reference's outputs (positions, faces, face_area, vertex_area, L^T).
 * Icosphere level (mesh.py:216-246), half-edge h = 3 f + e (edge e of face
 * f runs faces[f][e] -> faces[f][(e+1)%3]), twin = opposite half-edge or -1:
 *   ft_ico_flags      flag[h] = 1 where h is its edge's first encounter;
 *   ft_ico_midpoints  with incl = inclusive scan of the flags: mid[h] = the
 *                     midpoint id, new positions unit(p[u] + p[v]) written
 *                     at n_old.. (positions has room for them);
 *   ft_ico_children   the 4 child faces per face and their twins;
 *   ft_renormalize    positions /= norm(positions, axis=1) (final pass).
 * ft_torus_grid       gen_periodic_grid (mesh.py:168-199).
 * ft_face_geometry    face area / normal / barycenter and area/3 per face
 *                     (TriMesh, mesh.py:56-84); period = the 2x3 period
 *                     vectors or NULL, quarter_r2 = the squared quarter of
 *                     the shortest lattice offset (TriMesh._wrap).
 * ft_vertex_area      per-vertex sum of area/3 in (face, corner) order;
 *                     corner = flattened face-corner positions sorted stably
 *                     by vertex, ptr = per-vertex offsets into it.
 * ft_uniform_laplacian  L^T (ptr/idx/val_t, CSC) and L (same pattern, val)
 *                     from the sorted one-ring nptr/nidx (n_v + 1 / 2E). */
int ft_ico_flags(int64_t n_half, const int32_t* twin, int32_t* flag, void* stream);
int ft_ico_midpoints(int32_t n_faces, const int32_t* faces, const int32_t* twin, const int64_t* incl,
                     int32_t n_old, double* positions, int32_t* mid, void* stream);
int ft_ico_children(int32_t n_faces, const int32_t* faces, const int32_t* twin, const int32_t* mid,
                    int32_t* faces_out, int32_t* twin_out, void* stream);
int ft_renormalize(int32_t n, double* positions, void* stream);
int ft_torus_grid(int32_t nx, int32_t ny, double spacing, double* positions, int32_t* faces,
                  void* stream);
int ft_face_geometry(int32_t n_faces, const double* positions, const int32_t* faces,
                     const double* period, double quarter_r2, double* area, double* normal,
                     double* barycenter, double* third, void* stream);
int ft_vertex_area(int32_t n_v, const int64_t* ptr, const int64_t* corner, const double* third,
                   double* out, void* stream);
int ft_uniform_laplacian(int32_t n_v, const int64_t* nptr, const int32_t* nidx, int32_t* ptr,
                         int32_t* idx, double* val_t, double* val, void* stream);

/* -- host-side sequential steps (CPU, no stream) --------------------------- */
/* ft_wind_triangles: the consistent winding of m dual triangles (int32
 * [m][3], host memory, flipped in place) by the reference's depth-first walk
 * (dual.py:284-313): roots in index order, edges 0-1, 1-2, 2-0, the
 * triangles of an edge in ascending index. */
int ft_wind_triangles(int64_t m, int32_t* tris);

/* -- the reference's public sparse algebra (sparse.py:279-420) ------------ */
/* General-purpose versions of the operations the Euler step fuses, bitwise
 * equal to the numba kernels (values FT_F64 only).  spgemm C = A B is
 * expand-sort-compress:
 *   ft_spgemm_count   counts[p] = nnz(A(:, u)) for every entry p (row u) of
 *                     B, nnz_b = nnz(B) (spgemm_bounds, _kernels.py:14-23,
 *                     per entry: the work is parallel over B's entries);
 *   ft_spgemm_expand  with offsets = the exclusive scan of those counts,
 *                     every product A(r, u) B(u, j) with key j * n_rows(A) + r
 *                     at offsets[p].., in the reference's order (u ascending,
 *                     then r);
 *   (the caller sorts the keys with a STABLE sort, carrying the values)
 *   ft_segment_sums   the sequential sum of every run of equal keys (starts =
 *                     the first index of each run), first term assigned as in
 *                     spgemm_numeric (_kernels.py:26-62); the caller drops
 *                     exact zeros and builds col_ptr from the keys. */
int ft_spgemm_count(const ft_csc* a, const ft_csc* b, int64_t nnz_b, int64_t* counts, void* stream);
int ft_spgemm_expand(const ft_csc* a, const ft_csc* b, int64_t nnz_b, const int64_t* offsets,
                     int64_t* keys, double* vals, void* stream);
int ft_segment_sums(const double* vals, int64_t n, const int64_t* starts, int64_t n_seg,
                    double* sums, void* stream);
/* Interest skeleton of (phi, lt) (build_skeleton, sparse.py:345-371;
 * _kernels.py:96-150): skel_rows == NULL counts rows per column into
 * counts[n_cols]; then, with skel_ptr the caller's prefix sum, fills. */
int ft_skeleton(const ft_csc* phi, const ft_csc* lt, int32_t* counts, const int32_t* skel_ptr,
                int32_t* skel_rows, void* stream);
/* a's values on the skeleton pattern, explicit zeros elsewhere; bad_row[j] =
 * the last row of a nonzero of a outside the pattern, else -1
 * (expand_to_skeleton, sparse.py:374-396; _kernels.py:153-176). */
int ft_expand(const ft_csc* a, const int32_t* skel_ptr, const int32_t* skel_rows, double* out_vals,
              int32_t* bad_row, void* stream);
/* out = v * (1 / s) per column (s = the sequential column sum) when s > 0,
 * unchanged otherwise; sums[j] = s (normalize_columns, sparse.py:399-420). */
int ft_normalize_columns(const ft_csc* a, double* out_vals, double* sums, void* stream);

/* -- quality metrics ------------------------------------------------------ */
/* Distance from every point (n_points x 3 doubles) to the closest point of
 * the triangles (tri_a / tri_b / tri_c: n_tri x 3 doubles each, the
 * corners): the O(samples x triangles) core of the sampled Hausdorff metric.
 * Replaces _kernels.point_triangle_distances (_kernels.py:285-366) bitwise,
 * including its 1e300 initial minimum.  scratch: n_points uint64 (device).
 * All pointers device memory. */
int ft_point_triangle_distances(const double* points, int32_t n_points, const double* tri_a,
                                const double* tri_b, const double* tri_c, int32_t n_tri,
                                uint64_t* scratch, double* out, void* stream);

/* -- labels -------------------------------------------------------------- */
/* Per-vertex argmax cell id; ties -> lowest cell; the base row wins only
 * if strictly greater -> -1 (UNCLAIMED).  Replaces field.sharp_labels
 * (field.py:324-356).  labels: int64[n_cols]. */
int ft_labels(const ft_csc* phi, int32_t dtype, int64_t* labels, void* stream);

/* -- Lloyd step ---------------------------------------------------------- */
/* Faces per layer row: the pattern (and values) of the reference's
 * faces_by_cell product  M^T * PHI^T  (lloyd.py:21-28): face f is in row r
 * when sum_{v in f, ascending} PHI(r, v) != 0, faces ascending per row.
 * Two calls: cell_faces == NULL counts (cell_ptr[n_rows+1] filled, the
 * caller allocates cell_ptr[n_rows] entries), then the fill.  Rows below
 * min_row are skipped (min_row = 1: cells only).  scratch: int32[2*n_rows].
 * *big_flag (device) != 0 when a row holds more than 16384 faces and was
 * left unsorted (the caller sorts those segments).  PHI must be FT_F64. */
int ft_faces_by_cell(const ft_csc* phi, int32_t min_row, int32_t n_faces,
                     const int32_t* faces, int32_t* cell_ptr, int32_t* cell_faces,
                     double* cell_values, int32_t* scratch, int32_t* big_flag,
                     void* stream);

/* Per cell c (layer row c+1): approximate centroid and normal
 * (approx_centroid, lloyd.py:42-64) and the back-projected seed vertex
 * (backproject, lloyd.py:67-112), with numpy's exact reduction orders.
 * status[c]: 0 ok, 1 vanished, 2 degenerate, 3 null normal, 4 ray miss;
 * hit_vertex[c] = vertex id or -1.  period: the 2 lattice vectors of a
 * torus mesh as 6 doubles in HOST memory, or NULL.  seeds: int64[n_cells]
 * (device).  All other pointers are device memory. */
int ft_lloyd_centroids(const double* positions, int32_t n_vertices,
                       const int32_t* faces, int32_t n_faces,
                       const double* face_area, const double* face_bary,
                       const double* face_normal, const double* period,
                       int32_t n_cells, const int32_t* cell_ptr,
                       const int32_t* cell_faces, const int64_t* seeds,
                       double* point, double* normal, int32_t* status,
                       int32_t* hit_vertex, void* stream);

/* Back-projection alone (backproject, lloyd.py:67-112) from caller-given
 * points and unit normals (n_cells x 3 doubles, device): status[c] must be
 * 0 on entry to take part; returns 4 (miss) or the hit vertex as above. */
int ft_lloyd_backproject(const double* positions, int32_t n_vertices, const int32_t* faces,
                         int32_t n_faces, const double* period, int32_t n_cells,
                         const int32_t* cell_ptr, const int32_t* cell_faces, const double* point,
                         const double* normal, int32_t* status, int32_t* hit_vertex, void* stream);

/* Lloyd on a partitioned field: a rank's faces (ascending;
 * faces / geometry arrays indexed by the rank's face list, vertex ids
 * global) and the cells' face lists over them (ft_faces_by_cell on the
 * rank's local field).
 *   ft_lloyd_partials  per cell: face count, sum of areas, sum of area *
 *                      barycenter (periodic: unwrapped around the seed), sum
 *                      of area * normal -> sums[n_cells][8]; summed over the
 *                      ranks by an all-reduce;
 *   ft_lloyd_finish    point, unit normal and status (0 ok, 1 vanished, 2
 *                      degenerate, 3 null normal) from the reduced sums;
 *   ft_lloyd_backproject_keys  the back-projection over the rank's faces,
 *                      plus the cross-rank key of its best hit: |t| (inf on
 *                      a miss) and the global face id (face_ids[face]); the
 *                      ranks all-reduce min |t|, then the min face id among
 *                      the ties (np.argmin's first occurrence). */
int ft_lloyd_partials(const double* positions, int32_t n_vertices, const int32_t* faces, int32_t n_faces,
                      const double* face_area, const double* face_bary, const double* face_normal,
                      const double* period, int32_t n_cells, const int32_t* cell_ptr,
                      const int32_t* cell_faces, const int64_t* seeds, double* sums, void* stream);
int ft_lloyd_finish(int32_t n_cells, const double* sums, double* point, double* normal, int32_t* status,
                    void* stream);
int ft_lloyd_backproject_keys(const double* positions, int32_t n_vertices, const int32_t* faces,
                              int32_t n_faces, const double* period, int32_t n_cells,
                              const int32_t* cell_ptr, const int32_t* cell_faces, const int32_t* face_ids,
                              const double* point, const double* normal, int32_t* status,
                              int32_t* hit_vertex, double* best_abs_t, int64_t* best_face, void* stream);

/* -- dual-mesh adjacency products --------------------------------------- */
/* One pass over vertices and faces of a (FT_F64) field collects, as keys in
 * four device hash sets (capacity: a power of two; empty slot = ~0):
 *   set_v  A_v pairs i<j (key i*n_cells+j): cells sharing a vertex with
 *          phi >= threshold                          (dual.py:60-91)
 *   set_t  A_t pairs: cells sharing a face of B = PHIbar M   (dual.py:94-99)
 *   set_x  A_t pairs whose threshold isolines cross inside a shared face of
 *          positive area                             (dual.py:107-215)
 *   set_3  junction triples i<j<k (key (i*n+j)*n+k) of every face with >= 3
 *          cells                                     (dual.py:223-231)
 * n_faces == 0 computes set_v only.  *overflow (device): bit flags: 1 = a set
 * is full, 2 = a vertex/face carries more than 32 thresholded cells; bit 2
 * (4): some cell pair skipped a zero-area face or a non-finite value in the
 * crossing test (the reference warns there, dual.py:187-199). */
int ft_dual_products(const ft_csc* phi, int32_t n_faces, const int32_t* faces,
                     const double* face_area, double threshold, uint64_t* set_v,
                     uint64_t* set_t, uint64_t* set_x, uint64_t* set_3,
                     int64_t set_capacity, int32_t* overflow, void* stream);

/* Candidate triangles of the dual mesh: the 3-cliques i < j < k of a
 * symmetric cell adjacency in CSR (n rows, sorted, no diagonal) -- the
 * ring intersection of build_dual (dual.py:331-340).  Count pass: tris ==
 * NULL, counts[q] for every entry q (nonzero only for q = (i, j), j > i);
 * fill pass at offsets[q] (the caller's exclusive prefix sum) as int32
 * triples (i, j, k), k ascending. */
int ft_clique_triangles(int32_t n, const int32_t* ptr, const int32_t* idx, int64_t* counts,
                        const int64_t* offsets, int32_t* tris, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FIELDTESS_CUDA_H */
