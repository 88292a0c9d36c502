/*
 * ghsvd.h -- C ABI of the B200-native implicit Hari-Zimmermann J-GHSVD engine.
 *
 * Computes the generalized hyperbolic SVD (GSVD when J = I) of a complex128
 * factor pair (F, G) under a diagonal sign matrix J, i.e. the eigenpairs of the
 * Hermitian-definite pencil (H, S) = (F^* J F, G^* G) without forming H or S
 * (Novakovic, Singer, Singer, Hari, arXiv:1907.08560; cited as PAPER.md:<line>).
 *
 * Conventions (all entry points):
 *  - Matrices are column-major complex128 = two IEEE doubles (re, im), column
 *    stride `ld*` in complex elements.  Unless stated otherwise a pointer may be
 *    HOST or DEVICE memory (the library copies with cudaMemcpyDefault, so host
 *    pointers cost a PCIe transfer on the context stream).
 *  - The library never allocates device memory: the caller passes one device
 *    workspace of ghsvd_workspace_bytes() bytes to ghsvd_create() and keeps it
 *    alive until ghsvd_destroy().  The library owns no caller buffer after a
 *    call returns (inputs are copied into the workspace).
 *  - Every call is enqueued on opts.stream and returns after the stream has
 *    drained (the calls are synchronous w.r.t. the host).
 *  - Status: 0 = OK, > 0 = warning (results valid), < 0 = error; after an
 *    error ghsvd_last_error() describes it and the context stays usable for
 *    ghsvd_destroy() (and for a new set_factors/factor).
 *  - Call order: create -> (factor | set_factors) -> [reduce] -> [get_factors]
 *    -> sweep [-> sweep ...] -> extract -> destroy; a new factor / set_factors
 *    starts the next problem in the same context; [get_state] between sweeps, and
 *    [set_state] after the problem's factor / set_factors / reduce, checkpoint and
 *    restore a solve.  Out-of-order calls return GHSVD_E_STATE.
 */
#ifndef GHSVD_H
#define GHSVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ghsvd_ctx_s* ghsvd_ctx;

typedef enum {
  GHSVD_OK = 0,
  GHSVD_NOT_CONVERGED = 1,     /* warning: C_max sweeps reached; results still extractable */
  GHSVD_E_INVALID_ARG = -1,    /* null pointer, m < n, ld < rows, J entry not +-1, bad option */
  GHSVD_E_STATE = -2,          /* call order violated */
  GHSVD_E_CUDA = -3,           /* a CUDA runtime call failed (message in ghsvd_last_error) */
  GHSVD_E_NCCL = -4,           /* NCCL unavailable or a collective failed */
  GHSVD_E_WORKSPACE = -5,      /* workspace smaller than ghsvd_workspace_bytes() */
  GHSVD_E_INDEFINITE_S = -6,   /* s_pp <= 0 or |s_pq| >= 1 after prescaling (G rank-deficient) */
  GHSVD_E_RANK_DEFICIENT = -7, /* singular T_a / block pivot / degenerate JQR pivot */
  GHSVD_E_NONFINITE = -8       /* NaN/Inf met in a Gram or a transformation */
} ghsvd_status;

enum { GHSVD_POINTWISE = 0, GHSVD_BLOCKED_BO = 1, GHSVD_BLOCKED_FB = 2 };
/* Block orderings of the blocked variants (csrc/ordering.h).  ROUND_ROBIN: the circle
 * method over the block columns (Sec 6.3-6.4, reading C-11).  LEVEL3 and HIER (reading R2-5
 * of PAPER.md:1815-1824, Sec 6.4: the blocking principle "applied recursively further")
 * group the block columns into super_blocks = 2Q super blocks: LEVEL3 runs an outer circle
 * method over the super blocks and ONE inner block sweep over every super pair (a Level-3
 * pivot of 2 super blocks, block-oriented; block pairs inside a super block are visited in
 * every outer step); HIER visits every block pair once per sweep, grouped by super pair.
 * With one super pair per rank (super_blocks = 2 * world_size) block columns change rank
 * only between outer steps: 2Q - 1 exchanges per sweep instead of nblocks - 1. */
enum { GHSVD_ORDER_ROUND_ROBIN = 0, GHSVD_ORDER_LEVEL3 = 1, GHSVD_ORDER_HIER = 2 };
/* Transformation criterion, eq (6.12) PAPER.md:1552-1562.  RELATIVE (default):
 * |H_pq| >= eps sqrt(n) |H_pp|^(1/2) |H_qq|^(1/2) or |S_pq| >= eps sqrt(n) on the
 * prescaled pivot; LITERAL: |H_pq| >= (max|H_ii| eps sqrt(n)) min|H_ii| as printed. */
enum { GHSVD_CRIT_RELATIVE = 0, GHSVD_CRIT_LITERAL = 1 };

typedef struct {
  int device;          /* CUDA ordinal of this rank's GPU */
  void* stream;        /* cudaStream_t owned by the caller (e.g. a torch stream); NULL = legacy default */
  int world_size;      /* 1 for a single GPU */
  int rank;            /* 0 .. world_size-1 */
  const void* nccl_id; /* 128-byte ncclUniqueId shared by all ranks; NULL if world_size == 1.
                        * Loopback id (test transport): 16 bytes "GHSVD-LOOPBACK\0\0" then a
                        * 112-byte group key.  The world_size ranks are then contexts of ONE
                        * process on one device, each driven from its own host thread (every
                        * call is collective, as with NCCL); block columns and reductions move
                        * by device copies between the contexts' workspaces, ordered by CUDA
                        * events and a host barrier (600 s timeout -> GHSVD_E_NCCL).  It runs
                        * the multi-GPU schedule of the blocked sweep without several GPUs. */
  int variant;         /* GHSVD_POINTWISE | GHSVD_BLOCKED_BO | GHSVD_BLOCKED_FB */
  int ordering;        /* GHSVD_ORDER_* (blocked variants; the pointwise variant is round-robin only) */
  int nblocks;         /* blocked: number of block columns (even; 0 = auto); Sec 6.4.1 */
  int max_sweeps;      /* C_max, default 30 (Algorithm 2) */
  int criterion;       /* GHSVD_CRIT_RELATIVE | GHSVD_CRIT_LITERAL */
  double eps;          /* machine precision in (6.12); 0 => 2^-53 */
  int cluster;         /* pointwise: CTAs per column pair (0 = auto: kernel 2 uses 4 when m >= 4096,
                          else 1; kernels 1/3 the smallest cluster whose slices fit shared memory) */
  int threads;         /* pointwise: threads per CTA (0 = auto: kernel 2 with m >= 4096 uses 128) */
  int use_graph;       /* capture each sweep's steps in a CUDA graph (default 1) */
  int kernel;          /* pointwise step kernel: 0 = auto (= 2), 1 = one cluster per pair, TMA-staged slices;
                          2 = two-pass through L2 (default); 3 = persistent pipelined TMA */
  int detail_timing;   /* blocked: 1 = CUDA events around every kernel on its launching stream
                          (fills t_* in ghsvd_stats; kernels of the two halves overlap, so the spans
                          are upper bounds of the kernels' own durations); 2 = only around the F/G
                          updates of every 8th block step, the sampled phase rotating with the
                          sweep (every step if there are fewer than 16): t_update, t_update_fg,
                          flops_update_fg and launches_update_fg then cover ONLY those sampled
                          launches (t_gram, t_pivot stay 0), while flops_update covers all
                          (~0.1 % of the sweep time instead of ~1.2 % at 1 on config 3) */
  int want_x;          /* also accumulate W = Z'^{-1} during the sweep so that ghsvd_extract_x
                          can return X = Z^{-1} = Sigma Z'^{-1} (NEXT-1):
                          pointwise by 2x2 inverses, blocked by block-pivot inverses.
                          Costs one more n x n buffer and its updates.  Pointwise kernel 2 only. */
  int exchange_overlap;/* multi-GPU blocked exchange (Sec 6.4.3): 0 (default) = ONE communicator and
                          one grouped send/recv per block step on the context stream, moving the F, G
                          and Z', W block columns together after all updates of the step; 1 = two
                          communicators (ncclCommSplit) on two streams, the Z', W part leaving right
                          after the Z' update so the next step's Grams need not wait for it (the
                          paper's future-work overlap). */
  int schedule;        /* blocked schedule / arithmetic alternatives, bitmask of GHSVD_SCHED_* (0 = the
                          measured default; every schedule flag is bitwise-equal to it, the
                          arithmetic flags are tested against the oracle) */
  int groups;          /* blocked, one rank: >= 2 selects the pipelined pair-group schedule (0 = off) */
  int gram_splits;     /* blocked: row splits of the block Grams (0 = planned against wave quantization) */
  const char* trace_path; /* blocked: write the first sweep's launch timeline (first-CTA start,
                          last-CTA end per launch) as CSV to this path (NULL = off) */
  int super_blocks;    /* LEVEL3 / HIER orderings: number of super blocks, even, dividing the number of
                          block columns (HIER: an even number of block columns per super block, or 1);
                          0 = 2 * world_size; on one GPU 4, or one super block per block column (the
                          round-robin) when the automatic partition has fewer than 32 block columns */
} ghsvd_options;
/* ghsvd_options.schedule bits.  ghsvd_default_options seeds schedule, groups, gram_splits and
 * trace_path from the environment (GHSVD_SERIAL, GHSVD_PRIO=0, GHSVD_SPLIT_BND, GHSVD_GRAM3M=0,
 * GHSVD_UPD4M, GHSVD_PIVOT_CL, GHSVD_SPLIT_FACTOR, GHSVD_GROUPS, GHSVD_NSPLIT, GHSVD_TRACE) for the tools; the
 * library itself reads only the options it is given. */
enum {
  GHSVD_SCHED_SERIAL = 1,     /* every kernel alone on the context stream (isolated kernel timing) */
  GHSVD_SCHED_NO_PRIO = 2,    /* no stream priorities */
  GHSVD_SCHED_SPLIT_BND = 4,  /* boundary-pair / rest split of each half's F/G update */
  GHSVD_SCHED_GRAM4M = 8,     /* exact 4M block Grams (default: 3M) */
  GHSVD_SCHED_UPD4M = 16,     /* exact 4M block updates (default: 3M) */
  GHSVD_SCHED_PIVOT_CL = 32,  /* two-CTA cluster block pivots */
  GHSVD_SCHED_SPLIT_FACTOR = 64 /* block-pivot factorizations in their own launch (k_blk_factor)
                                   instead of the Gram launch's last CTAs */
};

typedef struct {
  int sweeps;                 /* sweeps performed */
  int converged;              /* 1: stopped because a sweep had no "big" transformation */
  uint64_t pairs_visited;     /* sweeps * n(n-1)/2 */
  uint64_t transforms_all;    /* transformations applied (small + big) */
  uint64_t transforms_big;    /* "big" transformations (cos phi or cos psi != 1) */
  double seconds;             /* device time of the sweep loop (CUDA events) */
  double kernel_seconds;      /* device time of the sweep kernels alone (per-sweep events) */
  uint64_t launches;          /* sweep-kernel launches issued (pointwise: sweeps * (n-1)) */
  uint64_t alg_bytes;         /* algorithmic HBM bytes of the sweeps: per transformed pair
                                 128m+64n, per skipped pair 64m */
  double alg_flops;           /* algorithmic FP64 flops (blocked: Hermitian block Grams + updates) */
  double t_gram, t_pivot, t_update, t_exchange;  /* blocked: summed device time per kernel kind
                                                    (CUDA events, only if opts.detail_timing) */
  double flops_gram, flops_update;               /* blocked: algorithmic flops of those kernels;
                                                    updates count only the block pairs whose
                                                    update ran (device count per block step) */
  double max_offdiag_last;    /* max scaled off-diagonal measure seen in the last sweep */
  uint64_t all_per_sweep[64]; /* per-sweep counters (first 64 sweeps) */
  uint64_t big_per_sweep[64];
  /* blocked, dominant kernel (k_blk_update over the F and G row tiles, medium-priority
     stream): launches, algorithmic flops, and their summed device time (CUDA events on
     the launching stream; only if opts.detail_timing).  The Z' row tiles run on a
     low-priority stream that fills idle SMs and are excluded here. */
  uint64_t launches_update_fg;
  double flops_update_fg, t_update_fg;
  /* blocked: the partition and ordering the sweep ran (block columns, super blocks of a
     LEVEL3 / HIER ordering (0: round-robin), block steps per sweep) */
  int nblocks, super_blocks, steps_per_sweep;
} ghsvd_stats;

/* Fill *opts with the defaults described above (device 0, world_size 1). */
void ghsvd_default_options(ghsvd_options* opts);

/* Device workspace needed for factors with at most m rows and n columns
 * (nl > 0: also room for ghsvd_factor with N_L = nl).  Returns 0 on bad args. */
size_t ghsvd_workspace_bytes(const ghsvd_options* opts, int64_t m, int64_t n, int64_t nl);

/* Create a context bound to opts->device/stream over a device workspace sized
 * by ghsvd_workspace_bytes(opts, m, n, nl).  *out is set on success. */
ghsvd_status ghsvd_create(const ghsvd_options* opts, int64_t m, int64_t n, int64_t nl,
                          void* workspace, size_t bytes, ghsvd_ctx* out);

/* Phase 1 (Algorithm 1; eqs 4.1-4.3):  per atom a,
 * T_a = [[TAA_a, TAB_a], [TAB_a^*, TBB_a]] (lower triangle read) is factored by
 * HEBPJ (Bunch-Parlett complete pivoting, Sec 4.2-4.3) into Mt_a^* Jt_a Mt_a,
 * F_a = Mt_a [A_a; B_a] and G_a = [A_a; U_a B_a].  A, B: NA blocks of NL x NG
 * (block a at offset a*NL*NG, ld NL); U: NA*NL reals; TAA, TAB, TBB: NA blocks
 * of NL x NL (ld NL).  m = 2*NA*NL and n = NG must fit the context.  The rows of
 * F are then stably sorted so that J = diag(I_{n+}, -I_{m-n+}) (Sec 4.5.1).
 * Errors: GHSVD_E_RANK_DEFICIENT if some T_a is numerically singular. */
ghsvd_status ghsvd_factor(ghsvd_ctx ctx, int64_t NA, int64_t NL, int64_t NG,
                          const void* A, const void* B, const double* U,
                          const void* TAA, const void* TAB, const void* TBB);

/* Direct entry: F, G are m x n (ld >= m), J has m entries of +-1 (int8).
 * F's rows are stably sorted by J (+ first); G is copied as is.  Odd n is
 * bordered by one row and column (Sec 6.3.2).  Errors: INVALID_ARG. */
ghsvd_status ghsvd_set_factors(ghsvd_ctx ctx, int64_t m, int64_t n, const void* F, int64_t ldf,
                               const int8_t* J, const void* G, int64_t ldg);

/* Optional Phase 2 (Sec 5, eq 5.1): JQR of F with diagonal + partial pivoting,
 * hyperbolic Householder reflectors and (J,I) URV 2x2 pivots; G prepermuted by
 * P2 and reduced by Householder QR (R kept, diag real >= 0).  Afterwards
 * m = n.  May follow a ghsvd_get_factors (which then exported the Phase-1
 * factors); at most once per problem, before ghsvd_sweep.
 * flags: 0, or GHSVD_REDUCE_COLPIV: the QR of G P2 with column pivoting by norm,
 * P4 (G P2) P5 = Q G', F' = F P5 (the "slower but more stable"
 * path for a badly conditioned G~; no row pivoting P4); the combined permutation
 * P2 P5 is what ghsvd_get_factors exports and ghsvd_extract undoes.
 * Default for m n^2 >= 2e10 (else unblocked; GHSVD_REDUCE_BLOCKED / _UNBLOCKED force either):
 * BLOCKED (NEXT-4, the paper's "blocking and delaying the columns updates",
 * PAPER.md:1271-1275): left-looking panels of <= 33 reflectors in the compact form
 * I + S T S^* J, the trailing columns updated once per panel by two ZGEMMs (cuBLAS,
 * loaded at run time).  The JQR's pivots are PLANNED on the J-Grammian H = F^* J F (formed
 * once by ZGEMM, its Schur complements updated per pivot): the paper's diagonal + partial
 * pivoting rule applied to H_k instead of to the columns (equal in exact arithmetic), each
 * planned pivot checked on the exact J-Grammian of its formed column(s) before use; the
 * first one off by more than a quarter (or of another inertia) hands over to the column
 * search.  GHSVD_REDUCE_COLSEARCH: the column search throughout (pivot searches on
 * downdated J-norms, exact at every panel start; a panel is cut when a formed pivot column
 * disagrees with its estimate).  The column-pivoted QR of G P2 plans its pivots likewise on
 * S = (G P2)^* (G P2) (diagonally pivoted Cholesky of its Schur complements, checked per
 * panel; GHSVD_REDUCE_COLSEARCH: the downdated-norm search).  The plain QR of G P2 of the
 * blocked form is cuSOLVER's ZGEQRF (loaded at run time; the paper's code calls LAPACK's
 * ZGEQR there), GHSVD_REDUCE_OWN_QR: this library's blocked Householder QR instead.
 * The pivot sequence may differ from the unblocked one on near-ties; the Grammians and
 * the pencil are preserved alike (tests).  GHSVD_REDUCE_UNBLOCKED: one reflector
 * application per column (round 1), also the fallback when cuBLAS cannot be loaded or
 * the n x n output-Z buffer cannot hold the panel (m > ~n^2 / 35).
 * Errors: GHSVD_E_RANK_DEFICIENT on a degenerate JQR pivot or rank-deficient G;
 * GHSVD_E_NONFINITE on non-finite J-norms; INVALID_ARG on unknown flags. */
enum { GHSVD_REDUCE_COLPIV = 1, GHSVD_REDUCE_UNBLOCKED = 2, GHSVD_REDUCE_BLOCKED = 4, GHSVD_REDUCE_COLSEARCH = 8,
       GHSVD_REDUCE_OWN_QR = 16 };
ghsvd_status ghsvd_reduce(ghsvd_ctx ctx, int flags);
/* After ghsvd_reduce: the first column whose planned JQR pivot the exact J-Grammian of its
 * formed column rejected (the column search continued from there); -1 if every planned
 * pivot was used; -2 if no planned JQR ran (unblocked form -- small problems, or when the
 * output-Z buffer cannot hold the panel --, or GHSVD_REDUCE_COLSEARCH).  No GPU work. */
int64_t ghsvd_reduce_fallback_col(ghsvd_ctx ctx);

/* Export the factors the sweep will start from (after factor/set_factors,
 * the J row sort, [reduce] and bordering): *m, *n (bordered sizes); F, G
 * (m x n, ld >= m) and J (m int8) if non-NULL; p2 (n int64, column j of the
 * current factors is column p2[j] of the Phase-1/set_factors factors) if
 * non-NULL.  Used so the CPU oracle runs on exactly the same bytes.  Before the first
 * sweep; a size-only query (F, J, G, p2 all NULL) is also allowed after sweeps. */
ghsvd_status ghsvd_get_factors(ghsvd_ctx ctx, int64_t* m, int64_t* n, void* F, int64_t ldf,
                               int8_t* J, void* G, int64_t ldg, int64_t* p2);

/* Phase 3: sweeps (Algorithm 2; Alg. 3 per step) until a
 * sweep has no "big" transformation (Sec 6.1.7) or C_max sweeps.  Z' starts at
 * I.  Returns GHSVD_OK or GHSVD_NOT_CONVERGED (warning) or an error; *out
 * (may be NULL) receives counters and device time of this call.  A further call
 * resumes from the current F', G', Z' (and W): a solve split into calls of C_max
 * sweeps each runs exactly the sweeps of one call with a larger C_max (bitwise
 * the same results; tests/test_gpu_resume.py).  Multi-rank: every rank calls it. */
ghsvd_status ghsvd_sweep(ghsvd_ctx ctx, ghsvd_stats* out);

/* Diagnostic: run only steps [s0, s0+ns) of the round-robin sweep on the current
 * factors (Z' initialised to I on the first call after factor/set_factors):
 * pointwise steps in [0, n-2], or for the blocked variants block steps in
 * [0, nblk-2] (single rank).  *all / *big receive the transformations applied. */
ghsvd_status ghsvd_run_steps(ghsvd_ctx ctx, int64_t s0, int64_t ns, uint64_t* all, uint64_t* big);

/* Outputs of Sec 6.1.7 and eq (3.2): for each column i,
 * lambda_i = (f_i^* J f_i) / (g_i^* g_i), sigma_f = Sigma'_F/Sigma,
 * sigma_g = Sigma'_G/Sigma, Z = Z' Sigma^-1 with rows un-permuted by P2
 * (Z~ = P2 Z); bordered column stripped.  Any output
 * pointer may be NULL.  Z is n x n (ldz >= n), complete on every rank (multi-rank: the
 * owners' columns are summed into every rank, see ghsvd_extract_local for the distributed
 * form).  col_ids (n int64) receives the global column index of each output column
 * (always the identity here). */
ghsvd_status ghsvd_extract(ghsvd_ctx ctx, double* lambda, double* sigma_f, double* sigma_g,
                           void* Z, int64_t ldz, int64_t* col_ids);

/* As ghsvd_extract, but Z stays DISTRIBUTED over the ranks: lambda,
 * sigma_f, sigma_g are complete on every rank (n each, combined over ranks), while Z
 * receives only the columns this rank owns after the sweep (the owner of block step 0),
 * packed: Z is n x *ncols (ldz >= n), col_ids[j] is the global column index of packed
 * column j (ascending within each block column), *ncols their count (ncols required; Z
 * requires col_ids; host or device pointers).  The union of the ranks' columns is each
 * column exactly once.  One rank: all n columns with identity ids.  Multi-rank: every
 * rank calls it (collective over lambda, Sigma). */
ghsvd_status ghsvd_extract_local(ghsvd_ctx ctx, double* lambda, double* sigma_f, double* sigma_g,
                                 void* Z, int64_t ldz, int64_t* col_ids, int64_t* ncols);

/* X = Z^{-1} = Sigma Z'^{-1}, the right generalized singular vectors of (3.1)
 * (F = U Sigma_F X, G = V Sigma_G X), with columns permuted back by P2
 * (X~ = X P2^T).  n x n (ldx >= n), host or device.  Requires opts.want_x and a
 * completed sweep; GHSVD_E_STATE otherwise. */
ghsvd_status ghsvd_extract_x(ghsvd_ctx ctx, void* X, int64_t ldx);

/* Checkpoint / restore of a solve in progress (between ghsvd_sweep calls).
 * ghsvd_get_state copies the sweep state -- F', G' (m x n, the bordered sizes
 * ghsvd_get_factors reports), Z' and, with opts.want_x, W = Z'^{-1} stored transposed
 * (n x n) -- to caller buffers (host or device; NULL = skip; W requires want_x).
 * ghsvd_set_state loads such a state into a context whose problem was set up the same
 * way (same factor/set_factors/reduce inputs, so J's row order, bordering and P2 agree;
 * state after factor/set_factors/reduce or a sweep); F, G, Z' are required, W iff
 * want_x.  The next ghsvd_sweep resumes from it: checkpoint after k sweeps, restore in
 * a new context (or process), and the remaining sweeps give bitwise the uninterrupted
 * result (tests/test_gpu_resume.py).  Multi-rank: every rank saves / restores its own. */
ghsvd_status ghsvd_get_state(ghsvd_ctx ctx, void* F, int64_t ldf, void* G, int64_t ldg, void* Zp,
                             int64_t ldz, void* W, int64_t ldw);
ghsvd_status ghsvd_set_state(ghsvd_ctx ctx, const void* F, int64_t ldf, const void* G, int64_t ldg,
                             const void* Zp, int64_t ldz, const void* W, int64_t ldw);

/* Copy the current transformed factors F', G' (m x n) to F, G (NULL = skip). */
ghsvd_status ghsvd_get_transformed(ghsvd_ctx ctx, void* F, int64_t ldf, void* G, int64_t ldg,
                                   void* Zp, int64_t ldz);

/* Test hook: evaluate the device 2x2 transformation (Sec 6.1, eqs 6.1-6.12)
 * on `count` pivots.  in: 8 doubles per pivot {hpp, hqq, hpq.re, hpq.im, spp,
 * sqq, spq.re, spq.im}; out: 8 doubles per pivot (z11, z21, z12, z22 complex,
 * Z' column-major); kind: int per pivot (0 skip, 1 identity, 2 small, 3 big,
 * < 0 error).  All three are DEVICE pointers.  tol = eps*sqrt(n). */
ghsvd_status ghsvd_hz2x2_batch(ghsvd_ctx ctx, int64_t count, const double* in, double tol,
                               int criterion, double* out, int* kind);

/* Multi-GPU helpers (blocked variant, Sec 6.4.3).  Host-only,
 * no GPU needed.  Rank r owns round-robin slots [r K, (r+1) K) of each block step,
 * K = nblk / (2 world).
 * ghsvd_block_owner: rank owning block column b in block step s (-1 on bad args).
 * ghsvd_exchange_plan: blocks `rank` sends (to send_peer) / receives (from recv_peer)
 *   between block steps s and s_next; arrays of nblk entries; 0 or -1.
 * ghsvd_nccl_unique_id: 128-byte ncclUniqueId for opts.nccl_id (rank 0 creates it and
 *   broadcasts it); 0, or -4 if NCCL cannot be loaded. */
int ghsvd_block_owner(int nblk, int world, int s, int b);
int ghsvd_exchange_plan(int nblk, int world, int rank, int s, int s_next, int64_t* send_blk,
                        int64_t* send_peer, int64_t* nsend, int64_t* recv_blk, int64_t* recv_peer,
                        int64_t* nrecv);
int ghsvd_nccl_unique_id(void* out128);
/* The same for any block ordering (ordering = GHSVD_ORDER_*, nsup = the resolved number of
 * super blocks, ignored for ROUND_ROBIN; see ghsvd_options.super_blocks).
 * ghsvd_order_steps: block steps per sweep (-1 on bad args).
 * ghsvd_order_pair: block pair (*p < *q) of slot k in block step s; 0 or -1.
 * ghsvd_block_owner_ord / ghsvd_exchange_plan_ord: as the round-robin forms above. */
int64_t ghsvd_order_steps(int ordering, int nblk, int nsup);
int ghsvd_order_pair(int ordering, int nblk, int nsup, int64_t s, int64_t k, int64_t* p, int64_t* q);
int ghsvd_block_owner_ord(int ordering, int nblk, int nsup, int world, int64_t s, int b);
int ghsvd_exchange_plan_ord(int ordering, int nblk, int nsup, int world, int rank, int64_t s, int64_t s_next,
                            int64_t* send_blk, int64_t* send_peer, int64_t* nsend, int64_t* recv_blk,
                            int64_t* recv_peer, int64_t* nrecv);

const char* ghsvd_last_error(ghsvd_ctx ctx);
void ghsvd_destroy(ghsvd_ctx ctx);

/* Library version string. */
const char* ghsvd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GHSVD_H */
