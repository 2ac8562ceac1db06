/* vreg_cuda.h -- thin C ABI between the C++ host layer (CudaEngine,
 * include/vreg_b200/) and the sm_100a kernels of libvreg_b200.so.
 *
 * Every entry point replaces one member (or free function) of the
 * reference's serial backend concept, cited as proj/<file>:<line> under
 * /root/reference (arxiv/paper_2008_12820). Plain pointers and sizes only:
 *
 *  - all field pointers are DEVICE pointers to float32, owned by the caller;
 *  - a scalar field holds the rank's x1-slab, n1_local*n2*n3 values, row-major
 *    with x3 innermost (grid.hpp:38-40); a vector field is ONE allocation of
 *    3 consecutive scalar fields (c1, c2, c3; field.hpp:25-36);
 *  - characteristics are stored as departure-point displacements in grid
 *    units, 3 scalar fields (disp = departure - node, per axis), plus an
 *    identity flag (engine.hpp:30-33, 111-155);
 *  - calls are ordered on the context's stream; scalar results are returned
 *    through host pointers after the stream reaches them;
 *  - errors never cross as exceptions: an int status (below), with the
 *    message from vreg_last_error(); the C++ layer rethrows the matching
 *    vreg exception type (types.hpp:19-41).
 */
#ifndef VREG_CUDA_H
#define VREG_CUDA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (types.hpp:17-41; exit codes via vreg_status_exit_code) */
enum {
  VREG_OK = 0,
  VREG_EPARAM = 2,     /* parameter_error  -> exit 2 */
  VREG_ENUMERICAL = 3, /* numerical_error  -> exit 3 */
  VREG_EIO = 4,        /* io_error         -> exit 4 */
  VREG_EINPUT = 5,     /* input_error (NaN coordinates, interp.cpp:43-44) */
  VREG_EDIM = 6,       /* dimension_error  -> exit 2 */
  VREG_ECONFIG = 7,    /* config_error     -> exit 2 */
  VREG_ECUDA = 8       /* device / runtime failure */
};

const char* vreg_last_error(void);
int vreg_status_exit_code(int status);

/* ---- grid (grid.hpp:13-64). Global sizes; the slab is derived from the
 * context's rank / world size (x1 split in equal contiguous slabs). */
typedef struct {
  int n1, n2, n3;
  int nt;
} vreg_grid;

typedef struct vreg_ctx_s* vreg_ctx;

/* Interpolation `degree` arguments: 1 trilinear, 3 cubic Lagrange (the
 * reference's two, interp.cpp:26-35), VREG_INTERP_BSPLINE3 cubic B-spline
 * on prefiltered coefficients (B200 extension named by the north star). */
#define VREG_INTERP_BSPLINE3 4

/* One context per GPU (per rank). EngineState analogue (engine.hpp:14-19):
 * stream, FFT plan cache keyed by grid, reduction scratch, memory pool,
 * kernel timers, NCCL communicator. */
int vreg_ctx_create(int device, vreg_ctx* out);
/* Multi-GPU: nccl_uid is the 128-byte ncclUniqueId from vreg_nccl_unique_id
 * on rank 0, broadcast by the caller. */
int vreg_nccl_unique_id(void* uid128);
int vreg_ctx_create_dist(int device, int rank, int nranks, const void* uid128,
                         vreg_ctx* out);
int vreg_ctx_destroy(vreg_ctx ctx);
int vreg_ctx_rank(vreg_ctx ctx, int* rank, int* nranks);
/* Pre-grow the device memory pool by up to `bytes` (capped at half the free
 * memory) so later allocations do not map fresh pages mid-solve. */
int vreg_ctx_reserve(vreg_ctx ctx, size_t bytes);
/* Host-only: the x1 halo plan for ghost width G on slabs of n1l planes
 * (G may exceed n1l: "wide" halos span several ranks; replaces the point
 * routing of SPEC.md:513-520 for far departure points). Chunk i (i < return
 * value <= cap) comes from the rank at ring distance d[i]: c[i] planes, the
 * owner's last c[i] planes into the lo ghost at plane lo[i], its first c[i]
 * planes into the hi ghost at plane hi[i]. Returns the chunk count, or -1. */
int vreg_halo_chunks(int n1l, int G, int cap, int* d, int* c, long long* lo, long long* hi);
/* Transpose (scatter) sweeps in exact fixed point: bitwise reproducible and
 * independent of the GPU count, ~10% slower matvec. Default off (fp32 L2
 * reductions, run-to-run differences in the last bits); env VREG_DETERMINISTIC=1. */
int vreg_ctx_set_deterministic(vreg_ctx ctx, int on);
/* Order of the regularisation operator A used by regop / inv_regop /
 * seminorm / h0_matvec / the GN matvec: 1 = H1, symbol |k|^2 (the
 * reference, spectral.cpp:61-63; default), 2 = H2, symbol |k|^4 (B200
 * extension named by the north star; no reference oracle -- analytic
 * single-mode checks in tests/test_gpu_h2.py). */
int vreg_ctx_set_reg_order(vreg_ctx ctx, int order);
/* The stream all calls on ctx are ordered on (cudaStream_t). */
int vreg_ctx_get_stream(vreg_ctx ctx, void** stream);
int vreg_ctx_set_stream(vreg_ctx ctx, void* cuda_stream);
void* vreg_ctx_stream(vreg_ctx ctx);
int vreg_ctx_synchronize(vreg_ctx ctx);
/* x1 slab of this rank for grid g: planes [offset, offset + n1_local). */
int vreg_slab(vreg_ctx ctx, const vreg_grid* g, int* n1_local, int* offset);
/* Kernel timers fft/fd/sl/ghost_comm/interp_comm/scatter_comm/scatter_buffer/
 * transpose_comm (counters.hpp:69-78), seconds, measured with CUDA events. */
int vreg_ctx_enable_timers(vreg_ctx ctx, int on);
int vreg_ctx_timers(vreg_ctx ctx, double out8[8]);
/* Per-kernel device time while timers are on: the idx-th named kernel
 * (sorted by name); returns VREG_EPARAM past the end. */
int vreg_ctx_kernel_stats(vreg_ctx ctx, int idx, char name64[64], uint64_t* count,
                          double* seconds);
int vreg_ctx_reset_kernel_stats(vreg_ctx ctx);
/* Communication volume per category (counters.hpp:49-59), bytes. */
int vreg_ctx_comm(vreg_ctx ctx, uint64_t out9[9]);
/* Number of kernel launches issued by this library since creation. */
int vreg_ctx_launches(vreg_ctx ctx, uint64_t* out);
/* SL tile boxes built so far and how many exceeded the shared-memory budget
 * (those tiles run the per-point global-memory path). */
int vreg_ctx_tile_stats(vreg_ctx ctx, uint64_t* tiles, uint64_t* misfit);

/* ---- stream-ordered pooled device memory (value-semantics churn, SURVEY
 * §7 hard part 6) */
int vreg_alloc(vreg_ctx ctx, size_t bytes, void** out);
int vreg_free(vreg_ctx ctx, void* p);
int vreg_memcpy_d2d(vreg_ctx ctx, void* dst, const void* src, size_t bytes);
int vreg_memcpy_h2d(vreg_ctx ctx, void* dst, const void* src, size_t bytes);
int vreg_memcpy_d2h(vreg_ctx ctx, void* dst, const void* src, size_t bytes);

/* ---- pointwise (field.hpp:67-141); ncomp = 1 (scalar) or 3 (vector) */
int vreg_fill(vreg_ctx, const vreg_grid*, int ncomp, float* x, double value);
int vreg_copy(vreg_ctx, const vreg_grid*, int ncomp, const float* x, float* y);
int vreg_axpy(vreg_ctx, const vreg_grid*, int ncomp, double a, const float* x, float* y);
int vreg_scale(vreg_ctx, const vreg_grid*, int ncomp, float* x, double a);
/* y = a*y + x (PCG direction update: scale then axpy, pcg.hpp:90-91) */
int vreg_aypx(vreg_ctx, const vreg_grid*, int ncomp, double a, const float* x, float* y);
int vreg_sub(vreg_ctx, const vreg_grid*, int ncomp, const float* a, const float* b, float* out);
int vreg_hadamard(vreg_ctx, const vreg_grid*, const float* a, const float* b, float* out);
int vreg_pointwise_dot(vreg_ctx, const vreg_grid*, const float* v3, const float* w3, float* out);
int vreg_axpy_scaled_vector(vreg_ctx, const vreg_grid*, double a, const float* s,
                            const float* w3, float* out3);

/* ---- reductions: plane-folded fp64 (field.hpp:143-188). Per-x1-plane
 * partials folded in global plane order, so results are bitwise
 * independent of the rank count. */
int vreg_inner(vreg_ctx, const vreg_grid*, int ncomp, const float* a, const float* b, double* out);
int vreg_max_abs(vreg_ctx, const vreg_grid*, int ncomp, const float* x, double* out);

/* ---- FD8 (fd.cpp:150-179; engine.hpp:77-82) */
int vreg_fd_grad(vreg_ctx, const vreg_grid*, const float* f, float* out3);
int vreg_fd_div(vreg_ctx, const vreg_grid*, const float* v3, float* out);

/* ---- semi-Lagrangian (engine.hpp:111-169; interp.cpp:39-123) */
/* RK2 characteristics of v: writes disp3, sets *identity = (max|v| == 0). */
int vreg_characteristics(vreg_ctx, const vreg_grid*, const float* v3, int degree,
                         float* disp3, int* identity);
/* out = I[f] at the departure points (interp_at). */
int vreg_interp(vreg_ctx, const vreg_grid*, const float* f, const float* disp3,
                int identity, int degree, float* out);
/* out = I^T z, the exact transpose of vreg_interp (scatter_at). */
int vreg_scatter(vreg_ctx, const vreg_grid*, const float* z, const float* disp3,
                 int identity, int degree, float* out);
/* Queries at arbitrary points in radians, interleaved xyz (interpolate,
 * interp.cpp:70-90), single GPU only; m points. */
int vreg_interp_points(vreg_ctx, const vreg_grid*, const float* f, const double* xyz,
                       int64_t m, int degree, float* out);
int vreg_scatter_points(vreg_ctx, const vreg_grid*, const double* xyz, const float* z,
                        int64_t m, int degree, float* acc);

/* ---- fused transport (transport.hpp:49-64, 90-228) */
/* m[t+1] = I[m[t]], t = 0..nt-1; m holds (nt+1) scalar fields, m[0] set. */
int vreg_solve_state(vreg_ctx, const vreg_grid*, const float* disp3, int identity,
                     int degree, float* m);
/* Incremental state m~_nt (transport.hpp:145-181) with the cached gradients
 * grads = (nt+1) vector fields; writes all slices mt[0..nt] when mt_all is
 * non-null, and the final slice to mt_final. */
int vreg_inc_state(vreg_ctx, const vreg_grid*, const float* disp3, int identity,
                   int degree, const float* grads, const float* vt3, float* mt_all,
                   float* mt_final);
/* out3 = sum_t w_t psi_t grad m_t, psi_nt = fin, psi_{t-1} = I^T psi_t
 * (transport.hpp:207-228). */
int vreg_transpose_assemble(vreg_ctx, const vreg_grid*, const float* disp3, int identity,
                            int degree, const float* grads, const float* fin, float* out3);
/* The GN Hessian matvec, HessianAdjoint::Transpose with the gradient cache
 * (optim.hpp:115-137): out3 = beta A vt + sum_t w_t psi_t grad m_t. */
int vreg_gn_matvec(vreg_ctx, const vreg_grid*, const float* disp3, int identity,
                   int degree, const float* grads, double beta, const float* vt3,
                   float* out3);
/* q = (1 + dt/2 D(dep_bwd)) / (1 - dt/2 D), D = div v (transport.hpp:49-64);
 * returns VREG_ENUMERICAL if dt/2 max|D| >= 0.99. */
int vreg_adjoint_source_factor(vreg_ctx, const vreg_grid*, const float* v3,
                               const float* disp_bwd3, int identity_bwd, int degree,
                               float* q);
/* lambda_t = I_bwd[lambda_{t+1}] .* q, lam holds nt+1 fields, lam[nt] set
 * (transport.hpp:106-121). */
int vreg_adjoint_sweep(vreg_ctx, const vreg_grid*, const float* disp_bwd3, int identity_bwd,
                       int degree, const float* q, float* lam);
/* out3 = sum_t w_t lam_t grad m_t (transport.hpp:184-201). */
int vreg_integrate_lambda_grad_m(vreg_ctx, const vreg_grid*, const float* lam,
                                 const float* grads, float* out3);

/* ---- spectral (spectral.cpp:48-288); FFTs on cuFFT, timed as "fft" */
int vreg_regop(vreg_ctx, const vreg_grid*, const float* v3, double beta, int unit_zero_mode,
               float* out3);
int vreg_inv_regop(vreg_ctx, const vreg_grid*, const float* v3, double beta, float* out3);
int vreg_seminorm(vreg_ctx, const vreg_grid*, const float* v3, double* out);
int vreg_leray(vreg_ctx, const vreg_grid*, const float* v3, float* out3);
/* fine grid g -> coarse grid g/2 (restrict) and back (prolong); ncomp 1|3 */
int vreg_restrict(vreg_ctx, const vreg_grid* fine, int ncomp, const float* f, float* out_coarse);
int vreg_prolong(vreg_ctx, const vreg_grid* fine, int ncomp, const float* fc, float* out_fine);
int vreg_high_pass(vreg_ctx, const vreg_grid*, int ncomp, const float* f, float* out);
/* H0 s = beta_pc A s (unit zero mode) + grad_mref (grad_mref . s)
 * (precond.hpp:30-42). */
/* Fused fine-grid steps of the two-level preconditioner (precond.hpp:143-160)
 * on one rank: begin writes rc3 = restrict(r3) and sc3 = restrict(InvA r3) on
 * the coarse grid (n/2) from ONE forward transform of r3 and keeps InvA r3's
 * spectrum; end writes out3 = prolong(sc3) + high_pass(InvA r3) with one
 * inverse transform. rc3 may be NULL (the split H0 solve starts from sc3
 * alone). VREG_ECONFIG on several ranks. */
int vreg_two_level_begin(vreg_ctx ctx, const vreg_grid* g, const float* r3, double beta_pc,
                         float* rc3, float* sc3);
int vreg_two_level_end(vreg_ctx ctx, const vreg_grid* g, const float* sc3, float* out3);

int vreg_h0_matvec(vreg_ctx, const vreg_grid*, const float* s3, const float* grad_mref3,
                   double beta_pc, float* out3);
/* Half-space spectrum of a scalar field, interleaved complex64,
 * n1 x n2 x (n3/2+1) (single GPU; test hook for fft.hpp:16-46). */
int vreg_fft_forward(vreg_ctx, const vreg_grid*, const float* f, float* out_c);

/* ---- synthetic inputs (syn.cpp:9-44) */
int vreg_syn_template(vreg_ctx, const vreg_grid*, float* m0);
int vreg_syn_velocity(vreg_ctx, const vreg_grid*, float* v3);

/* ---- slab distribution (engine.hpp:63-66 from_global/to_global): copy the
 * rank's slab out of / into a host array of the global field. */
int vreg_from_global(vreg_ctx, const vreg_grid*, int ncomp, const float* host_global,
                     float* dev_local);
int vreg_to_global(vreg_ctx, const vreg_grid*, int ncomp, const float* dev_local,
                   float* host_global);

#ifdef __cplusplus
}
#endif
#endif
