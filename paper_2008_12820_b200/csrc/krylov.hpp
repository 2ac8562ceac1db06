// Device-resident preconditioned CG (the solver of pcg.hpp:30-94 and of the
// H0 inner solves of precond.hpp:104-162), re-designed for the GPU:
//
//  * the iterate x, residual r and direction p are fp64 device vectors (the
//    reference's Real) -- fp32 for the inner H0 solves, whose tolerance is
//    eps_h0 eps_k; the operator and the preconditioner are fp32 device
//    callbacks, fed fp32 copies written by the fused update kernels;
//  * every scalar (rho, pq, alpha, beta, |r|, the stopping state, the
//    relative-residual history) lives in device memory: inner products are
//    per-x1-plane fp64 partials folded in global plane order on the device
//    (field.hpp:143-175 association, p-independent; all-gathered over NCCL
//    on several GPUs), and the fold kernels apply the CG recurrences;
//  * the loop is a CUDA graph with a conditional WHILE node whose body is
//    one iteration (precondition, direction, operator, step, test); the last
//    kernel of the body sets the loop condition, so a whole solve is one
//    graph launch with no host round trip per iteration. A solve issued
//    while the stream is being captured (the H0 inner solve inside the
//    outer body) becomes a nested conditional node.
//
// Iteration order (same decisions as pcg.hpp): the preconditioner is applied
// at the top of an iteration to the residual the previous one left, so a
// converged solve never applies it once more; negative curvature stops
// before the step (x unchanged, iteration not counted).
#pragma once

#include <functional>
#include <vector>

#include "common.cuh"

namespace vb {

struct KrylovState {
  double rho, pq, alpha, beta, rr, r0n, tol;
  int it, max_it, stop, conv, negcurv, pad;
};

struct KrylovStats {
  int iters = 0;
  double rel_res = 1;
  bool converged = false;
  bool negative_curvature = false;
  std::vector<double> history;  // relative residuals, [0] = 1 (0 if r0 = 0)
};

// stream-ordered device operation on ctx->stream: out3 = Op(in3), fp32
using KrylovOp = std::function<void(const float* in3, float* out3)>;

class Krylov {
 public:
  // fp64: iterates x, r, p in fp64 (the reference's Real); false: fp32
  // iterates (the operator then reads them in place)
  Krylov(vreg_ctx ctx, const Slab& s, bool fp64 = true);
  ~Krylov();
  Krylov(const Krylov&) = delete;
  Krylov& operator=(const Krylov&) = delete;

  // Solve A x = b. x (fp32, 3 components) holds the initial guess when x0,
  // the solution afterwards. Outside stream capture: runs (first iteration
  // eagerly, the rest as one conditional graph -- or one host-checked
  // iteration at a time when !graph or VREG_PCG_GRAPH=0) and returns the
  // statistics.
  // Inside a capture: records the solve into the captured graph and returns
  // empty statistics; `acc` (device, optional) then receives
  // acc[0] += iterations, acc[1] |= !converged when the graph runs.
  KrylovStats solve(const KrylovOp& A, const KrylovOp& M, const float* b, float* x, double tol,
                    int max_it, bool x0, unsigned long long* acc = nullptr, bool graph = true);

  // The H0 inner solve of precond.hpp:104-162 with the operator split
  // H0 = B + G (B = beta_pc A, G s = gm (gm . s), pointwise) and M = B^-1:
  // x holds x0 = M b on entry (the reference's initial guess), so r0 = -G x0;
  // y = B p and z = M r are carried by recurrences and an iteration applies
  // M once (to G p) instead of M and B. fp32 iterates only.
  KrylovStats solve_h0(const float* gm, const KrylovOp& M, const float* b, float* x, double tol,
                       int max_it, unsigned long long* acc = nullptr, bool graph = true);

  const Slab& slab() const { return s_; }
  bool fp64() const { return fp64_; }

 private:
  void issue_init(const KrylovOp& A, const float* b, const float* x, bool x0, double tol,
                  int max_it);
  void issue_body(const KrylovOp& A, const KrylovOp& M, unsigned long long cond);
  void issue_fold(int mode, unsigned long long cond);
  void issue_finish(float* x, unsigned long long* acc);
  void dot(const void* a, const float* b32, double* dst = nullptr);
  KrylovStats read_stats();
  void capture_loop(const KrylovOp& A, const KrylovOp& M, bool nested);

  vreg_ctx ctx_;
  Slab s_;
  int chunks_;
  size_t n3_;  // 3 N
  bool fp64_;
  void *x_ = nullptr, *r_ = nullptr, *p_ = nullptr;
  float *z32_ = nullptr, *q32_ = nullptr, *p32_ = nullptr, *r32_ = nullptr;
  double *part_ = nullptr, *part_all_ = nullptr;
  KrylovState* st_ = nullptr;
  double* hist_ = nullptr;
  int hist_cap_ = 0;
  KrylovState* h_st_ = nullptr;  // pinned
  cudaStream_t cap_stream_ = nullptr;
  // split H0 solve (solve_h0): gradient field, M, and the y / G p / M G p vectors
  const float* h0g_ = nullptr;
  const KrylovOp* h0m_ = nullptr;
  float *y_ = nullptr, *gp_ = nullptr, *mg_ = nullptr;
};

}  // namespace vb
