// internal.h -- context layout and helpers shared by the CUDA translation units
// of libghsvd (not part of the public ABI; see include/ghsvd.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ghsvd.h"

namespace ghsvd {

// Device-side counters of one sweep (a5): zeroed at sweep start, read back once.
struct DevCounters {
  unsigned long long all;      // transformations applied
  unsigned long long big;      // big transformations
  unsigned long long off_bits; // max scaled off-diagonal measure (non-negative double bits)
  int err;                     // sticky error (first negative kind seen), 0 = none
  int pad;
};

// Layout of the caller-provided workspace (all offsets 256-B aligned).
struct Layout {
  size_t off_F, off_G, off_Z, off_F2, off_G2, off_Z2, off_W, off_X, off_scr, off_misc, total;
  size_t scr_bytes;
};

struct Ctx {
  ghsvd_options o;
  std::string trace_path;     // owned copy of o.trace_path (o.trace_path points here)
  cudaStream_t stream;
  cudaStream_t cap_stream;    // private stream for graph capture
  cudaStream_t aux_stream;    // blocked: Z' updates overlapped with the next step
  cudaStream_t aux_stream2;   // blocked: second half of each step's block pairs
  std::vector<cudaStream_t> grp_streams;  // blocked, one GPU: one stream per pair group
  cudaStream_t hi_stream[2];  // blocked: high-priority streams of the latency-bound factor/pivot kernels
  cudaStream_t mid_stream[2]; // blocked: medium-priority streams of the Gram / F,G-update kernels
  char* ws;
  size_t ws_bytes;
  Layout L;
  int64_t m_cap, n_cap, nl_cap;  // capacity the workspace was sized for
  int64_t ldm, ldn;              // leading dimensions (rows of F/G and Z, padded)
  // current problem
  int state;                     // 0 created, 1 factors set, 2 swept
  int64_t m, n;                  // bordered sizes the sweep works on
  int64_t m_user, n_user;        // user sizes (before bordering)
  int64_t npos;                  // J = diag(I_npos, -I_{m-npos}) after the row sort
  bool bordered;
  bool z_init;                   // Z' set to I for the current factors
  bool have_p2;
  // device pointers into the workspace
  double2 *F, *G, *Z;            // current ("regular") factors
  double2 *F2, *G2, *Z2;         // Z2: extraction output / Phase 2 temporary (F2, G2 unused)
  double2* W;                    // want_x: W^T = (Z'^{-1})^T, updated like Z' (column pairs)
  double2* Xo;                   // want_x: X output of the extraction
  char* scr;                     // scratch
  DevCounters* cnt;
  int8_t* J;                     // m signs (sorted form) for export
  int64_t* p2;                   // n column permutation of Phase 2
  double* lam;                   // n outputs (device)
  double* sf;
  double* sg;
  int* rowdest;                  // m+1 row destinations (row sort)
  // pointwise launch configuration
  int pw_cluster, pw_threads;
  bool pw_pipe;
  int pw_kind;
  int64_t pw_nclusters;           // clusters launched per step
  size_t pw_smem;
  // graph cache
  cudaGraphExec_t graph;
  int64_t graph_n, graph_key;
  cudaEvent_t ev0, ev1, ev2, ev3;
  // blocked partition of the last blocked sweep (host copies)
  std::vector<int> blk_start, blk_width;
  int blk_nsup = 0;              // resolved super blocks of a LEVEL3 / HIER ordering (ordering.h)
  int64_t p2_fallback_col = -2;  // planned JQR: first column whose planned pivot was rejected (-1: none, -2: no plan)
  int64_t p2_fallback_qr = -1;   // planned column-pivoted QR: end of the panel with the first rejected pivot
  // multi-GPU
  void* comm;                    // ncclComm_t (opaque)
  void* cublas = nullptr;        // cublasHandle_t of the blocked Phase 2 (dlopen'ed cuBLAS), lazily
  void* cusolver = nullptr;      // cusolverDnHandle_t (blocked Phase 2's plain QR of G P2), lazily
  std::string err;
};

#define GH_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
      return GHSVD_E_CUDA;                                                         \
    }                                                                              \
  } while (0)

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// pointwise.cu
ghsvd_status pw_configure(Ctx* ctx);
ghsvd_status pw_run_steps(Ctx* ctx, int64_t s0, int64_t ns);
ghsvd_status pw_sweep_launch(Ctx* ctx);   // enqueue one full sweep (graph or launches)
// extract.cu
ghsvd_status launch_extract(Ctx* ctx);
ghsvd_status launch_hz2x2_batch(Ctx* ctx, int64_t count, const double* in, double tol,
                                int criterion, double* out, int* kind);
// factors.cu
ghsvd_status launch_set_identity(Ctx* ctx, double2* Z, int64_t ldz, int64_t n);
ghsvd_status launch_row_scatter(Ctx* ctx, const double2* src, int64_t lds, double2* dst,
                                int64_t ldd, const int* dest, int64_t rows, int64_t cols);
ghsvd_status launch_sort_dest(Ctx* ctx, const int8_t* Jin, int64_t m, bool border,
                              int* dest, int8_t* Jout, int64_t* npos_dev);
// phase1.cu
ghsvd_status phase1_factor(Ctx* ctx, int64_t NA, int64_t NL, int64_t NG, const void* A,
                           const void* B, const double* U, const void* TAA, const void* TAB,
                           const void* TBB);
size_t phase1_scratch_bytes(int64_t m, int64_t n, int64_t nl);
// phase2.cu
ghsvd_status phase2_reduce(Ctx* ctx, int flags);
void phase2_release(Ctx* ctx);
size_t phase2_scratch_bytes(int64_t m, int64_t n);
// blocked.cu
ghsvd_status blk_sweep(Ctx* ctx, ghsvd_stats* st);
ghsvd_status blk_run_steps(Ctx* ctx, int64_t s0, int64_t ns);
size_t blk_scratch_bytes(const ghsvd_options* o, int64_t m, int64_t n);
// comm.cpp
enum { XCH_FG = 1, XCH_ZW = 2 };   // parts of the block-column exchange
ghsvd_status comm_exchange(Ctx* ctx, int nblk, int s_now, int s_next, const int* bstart, const int* bwidth, int part,
                           cudaStream_t st);
ghsvd_status comm_allreduce_counters(Ctx* ctx, DevCounters* c);
bool comm_step_moves(const Ctx* ctx, int nblk, long long s, long long s_next);
void comm_owned_blocks(const Ctx* ctx, int nblk, std::vector<int>& blocks);
ghsvd_status comm_finalize_outputs(Ctx* ctx, int nblk, const int* bstart, const int* bwidth, double* lam,
                                   double* sf, double* sg, double2* Zout, int64_t ldz, double2* Xout);

}  // namespace ghsvd
