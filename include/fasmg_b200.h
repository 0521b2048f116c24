/*
 * fasmg_b200.h -- C ABI of libfasmg_b200.so, the B200 (sm_100a) native
 * FAS multigrid path of arXiv 2510.11152.
 *
 * Two layers, matching the two reference interfaces that this library
 * replaces:
 *
 *  (b1) the kernel ABI of the reference backend dispatcher
 *       (/root/reference/pkg/src/fasmg/kernels/__init__.py:37-98): the 16
 *       kernels by name, same argument order and meaning as
 *       kernels/numpy_backend.py, on DEVICE arrays.  Every array argument is
 *       (pointer to the core-view origin, int64 element strides[ndim]) --
 *       the core view of PKG/grid.py:199-208 where array index equals grid
 *       index.  Bounds are inclusive.  Kernels mutate in place.
 *
 *  (b2) the solver engine behind FasSolver (PKG/fas.py:63-181): create a
 *       solver for one hierarchy/location/BC/plan/coefficients, load p and f,
 *       run V-cycles (each optionally followed by the outer residual norm),
 *       store p back.  The engine runs on its own parity-blocked layout and
 *       replays the V-cycle as a CUDA graph.
 *
 * Conventions: every int-returning function returns 0 on success or a
 * FASMG_E* code; fasmg_last_error() gives the message (thread-local).
 * `stream` is a cudaStream_t (may be NULL only where noted).  No function
 * synchronizes the device unless documented.  Not thread-safe per engine.
 *
 * BC encoding (PKG/boundary.py:22-87): kinds[6] / vals[6] in face order
 * xlo, xhi, ylo, yhi, zlo, zhi; kind 0 = dirichlet (reflected; wall value on
 * an edge axis), 1 = neumann (copy), 2 = periodic.  Edge axis `ea`: -1 for
 * cell-centered, else 0/1/2 (Location.edge_axis, PKG/grid.py:37-41).
 */
#ifndef FASMG_B200_H
#define FASMG_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define FASMG_OK 0
#define FASMG_EINVAL 1001
#define FASMG_ECUDA 1002
#define FASMG_ENOMEM 1003
#define FASMG_ESTATE 1004

/* ---- runtime ------------------------------------------------------------ */
const char* fasmg_last_error(void);
int fasmg_last_error_code(void);
int fasmg_version(void);
int fasmg_compiled_arch(void);
int fasmg_device_count(int* n);
int fasmg_stream_create(void** stream);
int fasmg_stream_destroy(void* stream);
int fasmg_stream_synchronize(void* stream);
int fasmg_stream_wait(void* waiter, void* signaler);

/* ---- (b1) kernel ABI: KER/__init__.py:37-46, KER/numpy_backend.py ------- */
/* replaces gs_sweep_2d (KER/numpy_backend.py:27-44) */
int fasmg_gs_sweep_2d(double* p, const long* ps, const double* f, const long* fs, double b,
                      double h2, double denom, int ilo, int ihi, int jlo, int jhi, int ipar,
                      int jpar, void* stream);
/* replaces gs_sweep_3d (KER/numpy_backend.py:47-62) */
int fasmg_gs_sweep_3d(double* p, const long* ps, const double* f, const long* fs, double b,
                      double h2, double denom, int ilo, int ihi, int jlo, int jhi, int klo,
                      int khi, int ipar, int jpar, int kpar, void* stream);
/* replaces apply_op_2d / apply_op_3d (KER/numpy_backend.py:91-99) */
int fasmg_apply_op_2d(double* out, const long* os, const double* p, const long* ps, double a,
                      double b, double inv_h2, int ilo, int ihi, int jlo, int jhi, void* stream);
int fasmg_apply_op_3d(double* out, const long* os, const double* p, const long* ps, double a,
                      double b, double inv_h2, int ilo, int ihi, int jlo, int jhi, int klo,
                      int khi, void* stream);
/* replaces residual_2d / residual_3d (KER/numpy_backend.py:102-112) */
int fasmg_residual_2d(double* out, const long* os, const double* p, const long* ps,
                      const double* fsrc, const long* fs, double a, double b, double inv_h2,
                      int ilo, int ihi, int jlo, int jhi, void* stream);
int fasmg_residual_3d(double* out, const long* os, const double* p, const long* ps,
                      const double* fsrc, const long* fs, double a, double b, double inv_h2,
                      int ilo, int ihi, int jlo, int jhi, int klo, int khi, void* stream);
/* replaces restrict_cc_2d/3d, prolong_cc_2d/3d (KER/numpy_backend.py:119-155) */
int fasmg_restrict_cc_2d(const double* fine, const long* fs, double* coarse, const long* cs,
                         int m0, int n0, void* stream);
int fasmg_restrict_cc_3d(const double* fine, const long* fs, double* coarse, const long* cs,
                         int m0, int n0, int l0, void* stream);
int fasmg_prolong_cc_2d(const double* coarse, const long* cs, double* fine, const long* fs,
                        int m0, int n0, void* stream);
int fasmg_prolong_cc_3d(const double* coarse, const long* cs, double* fine, const long* fs,
                        int m0, int n0, int l0, void* stream);
/* replaces restrict_edge0_2d/3d, prolong_edge0_2d/3d (KER/numpy_backend.py:162-224);
 * callers pass edge-axis-first permuted strides as PKG/transfer.py:41-45 does */
int fasmg_restrict_edge0_2d(const double* fine, const long* fs, double* coarse,
                            const long* cs, int m0, int n0, void* stream);
int fasmg_restrict_edge0_3d(const double* fine, const long* fs, double* coarse,
                            const long* cs, int m0, int n0, int l0, void* stream);
int fasmg_prolong_edge0_2d(const double* coarse, const long* cs, double* fine,
                           const long* fs, int m0, int n0, void* stream);
int fasmg_prolong_edge0_3d(const double* coarse, const long* cs, double* fine,
                           const long* fs, int m0, int n0, int l0, void* stream);
/* replaces weno_deriv0_2d/3d (KER/numpy_backend.py:231-262); out and wind
 * are interior-shaped (ni, nj[, nk]); q is the full array view */
int fasmg_weno_deriv0_2d(double* out, const long* os, const double* q, const long* qs,
                         const double* wind, const long* ws, int ni, int nj, int oi, int oj,
                         double inv_2h, double eps, void* stream);
/* whole weno3_convect of component `target` in one pass (PKG/weno.py:54-91,
 * the winds of PKG/weno.py:26-51 evaluated in place): out = interior view
 * of the result; vel[a] = data pointer of component a (halo g), vst[3a+b]
 * its strides; ext = target interior extents */
int fasmg_weno_convect(double* out, const long* os, const double* const* vel, const long* vst,
                       int dim, int target, int g, const int* ext, double inv_2h, double eps,
                       void* stream);
int fasmg_weno_deriv0_3d(double* out, const long* os, const double* q, const long* qs,
                         const double* wind, const long* ws, int ni, int nj, int nk, int oi,
                         int oj, int ok, double inv_2h, double eps, void* stream);

/* ---- field-level helpers ------------------------------------------------ */
/* replaces fill_ghosts (PKG/boundary.py:90-107) on a C-contiguous data array
 * of a field with n[dim] cells, edge axis ea and halo `halo` */
int fasmg_fill_ghosts(double* data, int dim, const int* n, int ea, int halo, const int* kinds,
                      const double* vals, void* stream);
/* the same fill on one rank's axis-0 slab of a field (local C-contiguous
 * array with ext0 rows along axis 0, n[0] the slab's cells): sides flagged
 * in iface (bit 0 lo, bit 1 hi) are rank interfaces whose rows hold the
 * neighbour's interior values; they are completed along axes 1..d-1 only,
 * the boundary condition applies on global walls (ns_slab.py) */
int fasmg_fill_ghosts_slab(double* data, int dim, const int* n, int ea, int halo,
                           const int* kinds, const double* vals, int iface, int ext0,
                           void* stream);
/* np.sum of a (non-contiguous) interior view in numpy 2.3's buffered-reduce
 * order, used by the mean projection (PKG/fas.py:145,156); out[0] on device.
 * scratch >= prod(ext) doubles; sums >= fasmg_view_sum_chunks() doubles */
int fasmg_view_sum(const double* v, const long* vs, int dim, const int* ext, double* scratch,
                   double* sums, double* out, void* stream);
long fasmg_view_sum_chunks(int dim, const int* ext);
/* np.sum(vals * vals) of an interior view, the residual norm's sum of
 * squares (PKG/grid.py:235-249): numpy squares into a contiguous temporary
 * and sums it with ONE flat pairwise sum; reproduced bitwise.  out[0] on
 * device; scratch >= fasmg_view_sumsq_scratch() doubles. */
int fasmg_view_sumsq(const double* v, const long* vs, int dim, const int* ext, double* scratch,
                     double* out, void* stream);
long fasmg_view_sumsq_scratch(int dim, const int* ext);
/* Slab form of the same reduction (SURVEY.md section 8e item v): per-chunk
 * sums of an axis-0 slab `ext` of an interior view whose WHOLE extent is
 * `gext`, with numpy's chunk length for gext (fasmg_view_chunk_len); the
 * slab must hold whole chunks.  Ranks all-gather the sums in rank order and
 * total them in chunk order (fasmg_chunk_total, or the same sequential
 * adds on the host). */
int fasmg_view_chunk_sums(const double* v, const long* vs, int dim, const int* ext,
                          const int* gext, double* scratch, double* sums, void* stream);
long fasmg_view_chunk_len(int dim, const int* gext);
int fasmg_chunk_total(const double* sums, long nch, double* out, void* stream);
/* v -= total[0] / count over an interior view */
int fasmg_sub_mean(double* v, const long* vs, int dim, const int* ext, const double* total,
                   double count, void* stream);

/* staggered operators (PKG/stencil.py:114-156): gradient_axis into a
 * contiguous edge-interior array; divergence of component core views into a
 * cell interior view */
int fasmg_gradient_axis(const double* pcore, const long* ps, double* out, int dim,
                        const int* n, int axis, double inv_h, void* stream);
int fasmg_divergence(const double* const* comps, const long* cs, double* out, const long* os,
                     int dim, const int* n, double inv_h, void* stream);
/* projection-step elementwise ops (ns.py; op codes in fasmg_natural.cu NsOp)
 * and the 5/7-point Laplacian at a field's interior points */
int fasmg_ns_elem(int op, double* out, const long* os, const double* const* in,
                  const long* is, double s0, double s1, int dim, const int* ext, void* stream);
int fasmg_laplacian(double* out, const long* os, const double* pcore, const long* ps, int dim,
                    const int* m, double inv_h2, void* stream);

/* momentum source of one velocity component in one pass (NS driver,
 * Table 3/5 step 1): out = ((u - s0*conv) - s0*(p[x+e_axis]-p[x])*inv_h)
 * [+ s1*Lap(u)] for order 2; out/conv interior views, u/p core views */
int fasmg_ns_rhs(int order, double* out, const long* os, const double* ucore, const long* us,
                 const double* conv, const long* cs, const double* pcore, const long* ps,
                 int dim, int axis, const int* m, double s0, double s1, double inv_h,
                 double inv_h2, void* stream);

/* ---- (b2) solver engine: FasSolver (PKG/fas.py:63-162) ------------------ */
/* FasSolver.__init__ (PKG/fas.py:71-89): n[dim] finest cells, mesh_level
 * coarsenings, operator a*p - b*Lap(p) (PKG/stencil.py:21-38), smoothing
 * plan as class masks (bit c = parity class q0*4+q1*2+q2 in 3D, q0*2+q1 in
 * 2D; one mask per ghost-refresh group of make_plan, PKG/smoothers.py:87),
 * s smoothing steps per stage.  Returns NULL on error. */
void* fasmg_engine_create(int dim, const int* n, int ea, double dmin, double dmax,
                          int mesh_level, double a, double b, const int* kinds,
                          const double* vals, int nmasks, const unsigned* masks, int s,
                          void* stream);
void fasmg_engine_destroy(void* engine);
/* Engines that never run concurrently (the momentum and pressure solves of
 * one projection step) can share their level arrays: create them in one
 * arena.  An engine that finds another engine was the last user of the
 * arrays clears them on load (the state of a fresh engine), so results are
 * unchanged.  The arena lives until it and every engine in it are
 * released. */
void* fasmg_arena_create(void);
void fasmg_arena_release(void* arena);
void* fasmg_engine_create_in(int dim, const int* n, int ea, double dmin, double dmax,
                             int mesh_level, double a, double b, const int* kinds,
                             const double* vals, int nmasks, const unsigned* masks, int s,
                             void* stream, void* arena);
/* copy p and f (core views, strides) into the engine (enqueued on the
 * engine stream) */
int fasmg_engine_load(void* engine, const double* pcore, const long* ps, const double* fcore,
                      const long* fs);
/* write the solution interior back into a core view */
int fasmg_engine_store(void* engine, double* pcore, const long* ps);
/* run `count` V-cycles (PKG/fas.py:96-128); with_norm adds the outer
 * residual's sum of squares after each (PKG/fas.py:149-151) and returns the
 * last one in *sumsq after synchronizing; use_graph replays a captured
 * CUDA graph */
int fasmg_engine_run(void* engine, int count, int with_norm, double* sumsq, int use_graph);
int fasmg_engine_residual_sumsq(void* engine, double* sumsq);
/* kernels per captured V-cycle (with_norm 0/1), or per iteration of the
 * device solve loop (with_norm 2: V-cycle + norm + convergence test) */
long fasmg_engine_kernels_per_vcycle(void* engine, int with_norm);
/* mean duration (ms, CUDA events on the engine stream) of one smoothing
 * half-sweep launch on `level`, over `reps` launches */
int fasmg_engine_time_sweeps(void* engine, int level, int reps, double* ms);
int fasmg_engine_level_info(void* engine, int level, long* info);

/* ---- axis-0 slab decomposition -------------------
 * One engine per rank owns the slab `rank` of every level whose block-plane
 * count splits into >= min_planes (even) planes per rank; coarser levels are
 * replicated.  After each half-sweep the updated classes' boundary planes
 * are pushed into the neighbours' halo planes (peer stores over NVLink /
 * CUDA IPC, or same-device stores for virtual ranks) and published with
 * system-scope release/acquire counters; the first replicated level is
 * all-gathered; the residual sum is reduced in fixed rank order.  Cell-
 * centred fields, x not periodic. */
void* fasmg_engine_create_slab(int dim, const int* n, int ea, double dmin, double dmax,
                               int mesh_level, double a, double b, const int* kinds,
                               const double* vals, int nmasks, const unsigned* masks, int s,
                               void* stream, int nranks, int rank, int min_planes);
int fasmg_engine_export_count(void* engine);
/* device pointers of this engine: P[0..nl), F[0..nl), flags, allpart */
int fasmg_engine_export(void* engine, unsigned long long* out);
/* every rank's export arrays, concatenated, as pointers valid in this process */
int fasmg_engine_connect(void* engine, const unsigned long long* all, int nranks);
/* [first replicated level, local planes of level 0, global plane offset] */
int fasmg_engine_slab_info(void* engine, int* out);
/* push the level-0 halo planes after fasmg_engine_load */
int fasmg_engine_sync_halos(void* engine);
/* asynchronous run/result pair (ranks that must run concurrently) */
int fasmg_engine_launch(void* engine, int count, int with_norm);
/* capture + instantiate the V-cycle graph without launching it; every rank
 * sharing a device is prepared before any launches (lazy module loading
 * would otherwise wait on the peers' spin-waits) */
int fasmg_engine_prepare(void* engine, int with_norm);
/* the whole outer solve loop (PKG/fas.py:147-154) as ONE graph launch: up to
 * k_max V-cycles + norms on the loaded state, the convergence test
 * res = scale*sqrt(sumsq) <= tol evaluated on the device (a WHILE
 * conditional node); history (host, k_max doubles) and *iters out. */
int fasmg_engine_solve(void* engine, int k_max, double tol, double scale, double* history,
                       int* iters);
/* fasmg_engine_solve in two halves for slab ranks that must all be enqueued
 * before any is waited on (ranks on one device): capture the loop's graph on
 * every rank first (prepare_solve), then launch each, then wait each.  All
 * ranks see the same rank-ordered norm and stop together. */
int fasmg_engine_prepare_solve(void* engine);
int fasmg_engine_solve_launch(void* engine, int k_max, double tol, double scale);
int fasmg_engine_solve_wait(void* engine, double* history, int* iters);
/* self-test of the sweep kernels' reciprocal division: n random normal
 * numerators (|exponent| <= emax) x nd divisors; *bad = quotients whose bits
 * differ from IEEE division (expected 0) */
int fasmg_selftest_div(long n, unsigned long long seed, const double* dens, int nd, int emax,
                       unsigned long long* bad);
int fasmg_engine_result(void* engine, double* sumsq);
/* test access: level geometry [cls, s0, s1, E0, E1, E2, B0, off0, G0] and a
 * device copy of a level's blocked P (which=0) or F (which=1) arrays */
int fasmg_engine_level_geom(void* engine, int level, long* out);
int fasmg_engine_level_copy(void* engine, int level, int which, double* dst);
int fasmg_ipc_get_handle(void* ptr, unsigned char* out64);
int fasmg_ipc_open_handle(const unsigned char* in64, void** ptr);
int fasmg_ipc_close_handle(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* FASMG_B200_H */
