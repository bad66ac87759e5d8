/* moa.h — C ABI of the B200-native MoA Operational-Normal-Form GEMM (libmoa.so).
 *
 * Paper: L. Mullin et al., "From array algebra to energy efficiency on GPUs"
 * (arXiv 2306.11148); "P:n" = line n of PAPER.md. Design: DESIGN.md.
 *
 * Everything here is plain C: integers, raw pointers, opaque handles. No torch
 * types. All matrices are ROW-MAJOR and CONTIGUOUS ("generic row-major form",
 * P:77-82; "ALL arrays are accessed contiguously"):
 *     A<m,n>: element (i,k) at A[(i*n)+k];  B<n,p>: (k,j) at B[(k*p)+j];
 *     C<m,p>: (i,j) at C[(i*p)+j]            (Eq. 1; Eq. 3)
 *
 * Ownership: the caller owns every buffer. The library never allocates device
 * memory per call, never frees caller memory and never synchronises the
 * caller's stream (except moa_gemm_host, which is documented as synchronous).
 * The library owns only communicator handles (moa_comm_t) and a mutex-guarded
 * per-device cache of device properties.
 *
 * Errors: every entry point returns a moa_status. Argument validation happens
 * before any CUDA or NCCL call, so an invalid call has no side effect. CUDA
 * launch errors map to MOA_ERR_CUDA and NCCL errors to MOA_ERR_NCCL, with detail
 * in moa_last_error() (thread-local). Asynchronous device faults surface at the
 * caller's next synchronisation, as in CUDA. Nothing aborts or prints.
 */
#ifndef MOA_H
#define MOA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOA_ABI_VERSION 1

/* Element types. MOA_F64 is the paper's type (double).
 * MOA_F32: exact fp32, one IEEE fma per (i,j,k), k ascending.
 * MOA_F32_3XTF32: fp32 in/out via three TF32 tensor-core products
 *   (big*big + big*small + small*big); NOT exact, tolerance 5e-3 (north_star). */
typedef enum { MOA_F64 = 0, MOA_F32 = 1, MOA_F32_3XTF32 = 2 } moa_dtype;

typedef enum {
  MOA_OK = 0,
  MOA_ERR_INVALID_SHAPE = 1,   /* negative extent, overflow of m*n / n*p / m*p, bad partition */
  MOA_ERR_INVALID_DTYPE = 2,
  MOA_ERR_NULL_POINTER = 3,    /* NULL where the extents require memory */
  MOA_ERR_ALIASING = 4,        /* C overlaps A or B (":=" needs distinct output) */
  MOA_ERR_MISALIGNED = 5,      /* pointer not aligned to the element size */
  MOA_ERR_INVALID_INDEX = 6,   /* psi index out of bounds (0 <=* i <* rho xi) */
  MOA_ERR_CUDA = 7,
  MOA_ERR_NCCL = 8,
  MOA_ERR_UNSUPPORTED_DEVICE = 9, /* not an sm_100 device */
  MOA_ERR_NOT_REGISTERED = 10     /* pointer is not inside a window of the communicator */
} moa_status;

/* Kernels the static plan can choose. */
typedef enum {
  MOA_KERNEL_NONE = 0,          /* no work (m == 0 or p == 0) */
  MOA_KERNEL_ZERO_FILL = 1,     /* n == 0: C := 0 (empty sum) */
  MOA_KERNEL_DGEMM_TMA = 2,     /* K1: fp64 DMMA, TMA + mbarrier warp-specialised */
  MOA_KERNEL_DGEMM_GENERIC = 3, /* K2: fp64 DMMA, plain loads (odd n/p, unaligned) */
  MOA_KERNEL_SGEMM_FFMA = 4,    /* K3: exact fp32 FFMA */
  MOA_KERNEL_SGEMM_3XTF32 = 5,  /* K4: 3xTF32 on tcgen05 tensor cores */
  MOA_KERNEL_SGEMM_GENERIC = 6  /* K3g: exact fp32, plain loads (n/p not multiples of 4, unaligned) */
} moa_kernel;

/* Static block plan ("block sizes derived statically from shapes and types",
 * P:12-13; "make [sizel, sizer] as close as possible to the GPU cache sizes",
 * P:238-245). Pure function of (m, n, p, dtype, device properties); no
 * autotuning. bk and the k order depend only on dtype, never on m, so any row
 * block computed alone is bitwise equal to the same rows of the full product. */
typedef struct {
  int32_t kernel;        /* moa_kernel */
  int32_t bm, bn, bk;    /* CTA tile: the lifted block of C (bm x bn) and k-slab bk */
  int32_t stages;        /* shared-memory ring depth */
  int32_t threads;       /* threads per CTA */
  int32_t ctas_per_sm;   /* resident CTAs per SM the plan assumes */
  int32_t grid;          /* CTAs launched (persistent: min(tiles, sms*ctas_per_sm)) */
  int64_t tiles_m, tiles_n, tiles; /* ceil(m/bm), ceil(p/bn), product */
  int32_t raster_group;  /* tile-rows per rasterisation group (L2 reuse) */
  int32_t smem_bytes;    /* dynamic shared memory per CTA */
  int32_t sms;           /* SM count of the device planned for */
  int32_t reserved;
} moa_plan_t;

/* Opaque NCCL-backed communicator owned by the library. */
typedef struct moa_comm_s* moa_comm_t;

/* ------------------------------------------------------------------------
 * moa_gemm — C := A • B  (Eq. 3 / Eq. 5), ONF row-major contiguous.
 *   m, n, p : extents, >= 0 (rho A = <m,n>, rho B = <n,p>, rho C = <m,p>).
 *   A, B, C : DEVICE pointers of element type `dtype` (moa_dtype), row-major
 *             contiguous as above. C is overwritten (":=", reading R1); its
 *             byte range must not overlap A's or B's (MOA_ERR_ALIASING).
 *             Pointers must be aligned to the element size; 16-byte alignment
 *             with n, p even (f64) / multiples of 4 (f32) selects the TMA kernel,
 *             anything else the generic kernel (same results, bit for bit).
 *   stream  : cudaStream_t as void* (NULL = legacy default stream). Asynchronous.
 * m == 0 or p == 0: no-op. n == 0: C := 0 (cudaMemsetAsync).
 * Result (f64, f32): for every (i,j), the fma chain over k = 0..n-1 ascending
 * starting from +0 — i.e. Fig. 3 ip.c with its update contracted to
 * one fused multiply-add (reading R3), bitwise, for any finite inputs.
 * ------------------------------------------------------------------------ */
int moa_gemm(int64_t m, int64_t n, int64_t p, const void* A, const void* B, void* C, int dtype, void* stream);

/* moa_gemm with an explicit plan (from moa_plan, possibly edited: only bm/bn/
 * stages/raster_group/grid of a kernel-compatible plan are honoured). Used by the
 * block-size sweep (the paper's block-size experiment). Returns
 * MOA_ERR_INVALID_SHAPE if the plan is not valid for the shape/dtype. */
int moa_gemm_with_plan(int64_t m, int64_t n, int64_t p, const void* A, const void* B, void* C, int dtype,
                       const moa_plan_t* plan, void* stream);

/* moa_gemm_acc — the σ-blocked form with leading dimensions: C (+)= A • B for
 * row-major operands with row strides lda >= n, ldb >= p, ldc >= p (elements),
 * e.g. a column slice A[:, k0:k1] (lda = full n) and the contiguous row panel
 * B[k0:k1, :] (MoA order: one byte range).
 *   accumulate == 0: C := A • B (as moa_gemm);
 *   accumulate != 0: C := C + A • B, continuing every element's fma chain from the
 *   C in memory in k order — so a sequence of k-panel calls over ascending
 *   panels reproduces the one-call result bit for bit (f64, f32): "the sigma loop
 *   is broken up creating the block. This necessitates another addition loop to
 *   add up the blocks". (3xTF32: the prior C is added in the epilogue.)
 * Validation as moa_gemm, plus MOA_ERR_INVALID_SHAPE for a leading dimension
 * smaller than its row length; aliasing is checked on the strided byte spans. */
int moa_gemm_acc(int64_t m, int64_t n, int64_t p, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                 int64_t ldc, int accumulate, int dtype, void* stream);

/* moa_gemm_host — end-to-end call on HOST buffers: copies A_host and B_host into
 * the caller's device buffers A_dev/B_dev, runs the GEMM into C_dev, copies C_dev
 * back to C_host, and returns when C_host is complete (synchronous). Pipelined by
 * row lifting: B goes first, then A in row panels on a library-owned
 * copy stream; each panel's GEMM runs on `stream` as soon as its rows arrive and
 * its C rows stream back on a second copy stream, so H2D, compute and D2H overlap.
 * Bitwise identical to copy + moa_gemm + copy (for MOA_F32_3XTF32, B is not split
 * into k-panels, so this holds for every dtype). Host buffers should be pinned.
 * Same validation as moa_gemm on the device buffers; host pointers must be
 * non-NULL when their extents are non-zero. */
int moa_gemm_host(int64_t m, int64_t n, int64_t p, const void* A_host, const void* B_host, void* C_host,
                  void* A_dev, void* B_dev, void* C_dev, int dtype, void* stream);

/* moa_gemm_lifted_host — moa_gemm_host for the row-lifted product (COLLECTIVE;
 * dimension lifting of the i loop, Fig. 4 ip_rows.c P:150-171; every
 * processor reads all of B, P:165 / reading R13):
 * rank g's rows [row0_g, row0_g + rows_g) = moa_lift_rows(m, G, g).
 *   A_host, C_host : rank g's rows_g x n / rows_g x p HOST rows (pinned);
 *   B_host         : n x p HOST matrix on rank 0, ignored (may be NULL) elsewhere;
 *   A_dev, B_dev, C_dev : device buffers of rows_g x n, n x p, rows_g x p.
 * Same pipeline as moa_gemm_host; B's k-panels cross the host link on rank 0 only
 * and reach every rank by one NCCL broadcast per panel on the communicator's side
 * stream, so B's host copy, its broadcast and the first row panel's compute
 * overlap. Synchronous. Bitwise equal to moa_gemm on the rank's rows. */
int moa_gemm_lifted_host(int64_t m, int64_t n, int64_t p, const void* A_host, const void* B_host, void* C_host,
                         void* A_dev, void* B_dev, void* C_dev, int dtype, void* stream, moa_comm_t comm);

/* ------------------------------------------------------------------------
 * moa_gemm_lifted — row-lifted C := A • B over the communicator's G ranks
 * (dimension lifting of the i loop onto processors, Fig. 4
 * ip_rows.c P:150-171). COLLECTIVE: every rank calls it with identical m, n, p,
 * dtype. Rank g owns rows [row0_g, row0_g + rows_g) of A and C, with
 * (row0_g, rows_g) = moa_lift_rows(m, G, g).
 *   A_local : device, rows_g x n (rank g's rows of A).
 *   B       : device, n x p on every rank; input on rank 0, overwritten with
 *             rank 0's B on the others (in-place ncclBroadcast over NVLink —
 *             every processor needs all of B: B carries no processor index in
 *             ip_rows.c; reading R13).
 *   C_local : device, rows_g x p, receives rank g's rows of C.
 *   C_full  : NULL, or a device m x p buffer that receives all of C on every
 *             rank (gather, reading R14).
 * Bitwise identical to moa_gemm on one GPU (row-block invariance of the plan).
 * If B lies inside a window from moa_comm_alloc_window (every rank passes its own
 * copy), the exchange is copy-engine pulls instead of NCCL broadcasts
 * (MOA_XF_PULL_B in moa_exchange_plan): after an entry barrier every rank g > 0
 * reads B's k-panels (moa_pull_panels) from rank 0's copy over NVLink into its
 * own, on a side stream, and the compute of panel j waits only for panel j; no SM
 * is taken from the GEMM. Rank 0 computes its rows in one launch. An exit barrier
 * keeps rank 0's B unchanged until every pull is complete.
 * Errors: checks that depend only on (m, n, p, dtype, G, npanels) fail identically
 * on every rank before any collective. Checks of THIS rank's pointers (NULL,
 * alignment, overlap) can fail on one rank only; that rank returns before any
 * collective while its peers block in the first one — as with NCCL, any error
 * from a collective call is fatal for the communicator (destroy it on every rank).
 * moa_comm_agree lets a caller make the local checks collective first.
 * ------------------------------------------------------------------------ */
int moa_gemm_lifted(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_local, void* C_full,
                    int dtype, void* stream, moa_comm_t comm);

/* moa_gemm_lifted_direct — row lifting with NO copy of B.
 * COLLECTIVE. B must lie inside a window from moa_comm_alloc_window on every rank
 * (only rank 0's copy is read; the others are never written). Every rank's K1
 * producer streams B's k-slabs by TMA straight from rank 0's copy through this
 * process's NVLink mapping of rank 0's window — the broadcast disappears into the
 * GEMM's own loads. Entry barrier (rank 0's B is final), exit barrier (every read of
 * it is complete); C_full as moa_gemm_lifted. Bitwise identical to moa_gemm. Peer
 * reads do not stay in the reader's L2, so every tile row re-reads its B panel over
 * NVLink: a design alternative to the pulled copy, not the default.
 * Errors as moa_gemm_lifted; MOA_ERR_NOT_REGISTERED if B is not inside a window. */
int moa_gemm_lifted_direct(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_local,
                           void* C_full, int dtype, void* stream, moa_comm_t comm);

/* moa_gemm_lifted_ex — as moa_gemm_lifted with an explicit number of k-panels
 * (0 = the static choice moa_lift_panels). With npanels > 1 the broadcast of B
 * is pipelined: B's rows are split into npanels contiguous k-panels (each one
 * byte range in MoA row-major order), broadcast one after the other on a
 * library-owned side stream, and the rank's compute for panel j (moa_gemm_acc,
 * accumulate for j > 0) waits only for panel j — the exchange overlaps the
 * lifted compute. Results are bitwise identical to npanels = 1 for MOA_F64 and
 * MOA_F32 (for MOA_F32_3XTF32 they agree within its tolerance). 1 <= npanels <= 16. */
int moa_gemm_lifted_ex(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_local, void* C_full,
                       int dtype, void* stream, moa_comm_t comm, int npanels);

/* moa_gemm_lifted_cols — dimension lifting of the COLUMNS (j axis) across ranks:
 * Fig. 5 ip_cols.c at GPU level, "Dimension lifting over the columns of
 * B reveals parallelism also". COLLECTIVE. Rank g owns columns
 * [col0_g, col0_g + cols_g) = moa_lift_rows(p, G, g) of B and C.
 *   A       : device, m x n on every rank; input on rank 0, overwritten with rank
 *             0's A elsewhere (in-place broadcast: ip_cols.c reads A with no
 *             column-group index).
 *   B_local : device, n x cols_g, row-major contiguous (rank g's column block of B).
 *   C_local : device, m x cols_g, receives rank g's column block of C.
 *   C_full  : NULL, or device m x p receiving all of C on every rank; then
 *   workspace must hold m * ceil(p / G) elements (not needed when G == 1).
 *   If C_full lies inside a window from moa_comm_alloc_window (any dtype), the gather
 *   is fused into the GEMM epilogue instead (each rank's
 *   column block is computed into its columns of C_full, row stride p, and stored
 *   by the same epilogue into every peer's C_full; entry/exit barriers as in
 *   moa_gemm_lifted_gather); workspace is then unused.
 * Bitwise identical to moa_gemm on one GPU (the k order of every element is
 * unchanged by a j split). */
int moa_gemm_lifted_cols(int64_t m, int64_t n, int64_t p, void* A, const void* B_local, void* C_local, void* C_full,
                         void* workspace, int dtype, void* stream, moa_comm_t comm);

/* moa_gemm_lifted_2d — 2-D dimension lifting: the i axis over grid_rows and the j axis
 * over grid_cols (grid_rows * grid_cols = G; rank = r * grid_cols + c). COLLECTIVE.
 * Rank (r, c) owns rows [row0_r, row0_r + rows_r) = moa_lift_rows(m, grid_rows, r)
 * and columns [col0_c, col0_c + cols_c) = moa_lift_rows(p, grid_cols, c):
 *   A_panel : device, rows_r x n — input on (r, 0), broadcast along the process row;
 *   B_panel : device, n x cols_c — input on (0, c), broadcast along the process column;
 *   C_block : device, rows_r x cols_c, receives C[rows, cols].
 * Row and column sub-communicators are split from `comm` (ncclCommSplit) on first
 * use of a grid shape and cached in the communicator. Bitwise equal to one GPU. */
int moa_gemm_lifted_2d(int64_t m, int64_t n, int64_t p, int grid_rows, int grid_cols, void* A_panel, void* B_panel,
                       void* C_block, int dtype, void* stream, moa_comm_t comm);

/* moa_gemm_lifted_2d_gather — moa_gemm_lifted_2d with the all-gather of C fused into
 * the GEMM epilogue (as moa_gemm_lifted_gather): C_full (m x p, inside a window from
 * moa_comm_alloc_window on every rank; MOA_ERR_NOT_REGISTERED otherwise) receives
 * all of C on every rank. Rank (r, c) computes its block straight into C_full at
 * rows [row0_r, row0_r + rows_r) x columns [col0_c, col0_c + cols_c) (row stride p);
 * the same epilogue stores it into every other rank's C_full; C_block also receives
 * the block. Entry/exit barriers as moa_gemm_lifted_gather. Any dtype (the 3xTF32 kernel
 * carries the same epilogue). */
int moa_gemm_lifted_2d_gather(int64_t m, int64_t n, int64_t p, int grid_rows, int grid_cols, void* A_panel,
                              void* B_panel, void* C_block, void* C_full, int dtype, void* stream, moa_comm_t comm);

/* ------------------------------------------------------------------------
 * The row-lifted GEMM with the all-gather of C FUSED into the GEMM (SURVEY §8(f)
 * NEXT-1 step 3). Rows of C depend only on the same rows of A and all of B (Fig. 1,
 * P:90-99), so rank g's rows (Fig. 4 ip_rows.c P:150-171) are final as
 * soon as its tiles are; the gather (reading R14: every rank ends with all of C)
 * only places them. Instead of a GEMM
 * followed by ncclAllGather, the epilogue of the GEMM kernel stores every final C
 * tile of rank g's rows [row0_g, row0_g + rows_g) both into its own C_full and,
 * over NVLink, into every other rank's C_full at the same rows — so the exchange
 * of C overlaps the remaining tiles' tensor-core work instead of following it.
 *
 * moa_gemm_scatter — the epilogue on its own (usable on one GPU): moa_gemm_acc
 * (same arguments, same result in C), and every final C tile is also written to
 * dst[0..ndst): each an m x p row-major block with row stride ldc (DEVICE address;
 * may be a peer GPU's memory mapped into this process, e.g. from
 * moa_comm_window_peer). Every destination receives exactly the bits of C. With
 * accumulate != 0 (the last k-panel of a chain) only C is read. Any dtype: every kernel
 * carries the epilogue (for MOA_F32_3XTF32 the destinations receive exactly the bits of
 * C, which is within that variant's tolerance); 0 <= ndst <= 8 (MOA_ERR_INVALID_SHAPE); destinations
 * non-NULL when m*p > 0, aligned to the element size (MOA_ERR_MISALIGNED otherwise),
 * and disjoint from A, B, C and each other (MOA_ERR_ALIASING). A destination that is
 * not 16-byte aligned routes the call to the generic kernel (same bits; the TMA
 * kernels' epilogue uses 16-byte stores). Asynchronous on `stream`. */
int moa_gemm_scatter(int64_t m, int64_t n, int64_t p, const void* A, int64_t lda, const void* B, int64_t ldb,
                     void* C, int64_t ldc, int accumulate, int ndst, void* const* dst, int dtype, void* stream);

/* moa_comm_alloc_window — COLLECTIVE (every rank, same bytes): allocate `bytes` of
 * device memory on each rank with ncclMemAlloc and register it on the
 * communicator as an NCCL symmetric window (NCCL_WIN_COLL_SYMMETRIC), so every
 * rank's copy is load/store-reachable from every GPU; *ptr = this rank's copy.
 * The library owns the memory until moa_comm_free_window (COLLECTIVE) or
 * moa_comm_destroy; both synchronise the device first (no kernel may still be
 * storing into a window being released). MOA_ERR_NCCL if not every rank is in the NVLink
 * load/store domain (NCCL's LSA team) or registration fails.
 * moa_comm_window_peer — *out = this process's address of rank `peer`'s copy of
 * the window byte that `ptr` addresses in this rank's copy (for peer == rank, an
 * alias of ptr's memory at another virtual address; MOA_ERR_NOT_REGISTERED
 * if ptr is not inside a window; MOA_ERR_INVALID_INDEX for a bad peer). */
int moa_comm_alloc_window(moa_comm_t comm, size_t bytes, void** ptr);
int moa_comm_free_window(moa_comm_t comm, void* ptr);
int moa_comm_window_peer(moa_comm_t comm, const void* ptr, int peer, void** out);

/* moa_gemm_lifted_gather — row-lifted C := A • B with the fused gather. COLLECTIVE.
 *   A_local, B, m, n, p, npanels: as moa_gemm_lifted_ex (B broadcast from rank 0).
 *   C_full : m x p, inside a window from moa_comm_alloc_window on every rank
 *            (MOA_ERR_NOT_REGISTERED otherwise). On return (stream order) every
 *            rank's C_full holds all of C, bitwise equal to moa_gemm on one GPU.
 * Stream order: a one-element all-reduce barrier before the GEMM (no rank stores
 * into a peer's C_full before that peer reached this call) and one after it (all
 * peer stores are complete). Any dtype (for MOA_F32_3XTF32 with npanels > 1 the panel
 * sums are added in the epilogue, so C_full agrees with moa_gemm within that variant's
 * tolerance rather than bitwise); at most 9 ranks (one NVLink node). */
int moa_gemm_lifted_gather(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_full, int dtype,
                           void* stream, moa_comm_t comm, int npanels);

/* moa_lift_panels — static k-panel count for the lifted exchange: 1 when B does
 * not travel (nranks == 1), else ceil(bytes(B) / 512 MiB) clamped to [1, 8] and
 * to n/64. Pure function. */
int moa_lift_panels(int64_t n, int64_t p, int dtype, int nranks);

/* ------------------------------------------------------------------------
 * The exchange plan of the lifted paths (row a7 of the build; P:147-148, P:165,
 * P:188): the static, ordered list of collectives a lifted call issues on each
 * rank. It is a pure function of (variant, m, n, p, dtype, G, rank, grid, npanels,
 * flags) — the executors of moa_gemm_lifted*, _cols, _2d and _host walk exactly this
 * list — so ranks issue identical sequences (per communicator) by construction,
 * and the bytes each call moves can be checked against the model without a GPU.
 *   op      : MOA_COLL_BROADCAST (NCCL, in place unless noted), MOA_COLL_ALLGATHER
 *             (NCCL), MOA_COLL_BARRIER (one-int NCCL all-reduce on the stream),
 *             MOA_COLL_PULL (copy-engine read of `count` elements of rank `root`'s
 *             symmetric window over NVLink into this rank's copy; no SMs, no NCCL);
 *   comm    : which communicator carries it (world, the CTA-limited pipe split,
 *             the 2-D row / column splits);
 *   root    : broadcast root / pull source, as a rank of `comm`; -1 otherwise;
 *   group   : ops with the same group id > 0 are issued in one ncclGroupStart/End;
 *   operand : what travels (MOA_OPERAND_A, _B, _C);
 *   phase   : 0 before the compute, 1 overlapped with it (k-panels of B: the
 *             compute of panel `panel` waits for this op), 2 after it;
 *   offset, count : the data's element offset in the destination operand, and its
 *             element count (all-gather: each rank's send count).
 * Ops on a 1-rank communicator are never issued, so G == 1 plans are empty. */
typedef enum { MOA_COLL_BROADCAST = 1, MOA_COLL_ALLGATHER = 2, MOA_COLL_BARRIER = 3, MOA_COLL_PULL = 4 } moa_coll_op;
typedef enum { MOA_COMM_WORLD = 0, MOA_COMM_PIPE = 1, MOA_COMM_ROW = 2, MOA_COMM_COL = 3 } moa_comm_kind;
typedef enum { MOA_OPERAND_A = 0, MOA_OPERAND_B = 1, MOA_OPERAND_C = 2 } moa_operand;
typedef enum {
  MOA_XPLAN_ROWS = 0,      /* moa_gemm_lifted_ex / moa_gemm_lifted_gather */
  MOA_XPLAN_ROWS_HOST = 1, /* moa_gemm_lifted_host */
  MOA_XPLAN_COLS = 2,      /* moa_gemm_lifted_cols */
  MOA_XPLAN_2D = 3         /* moa_gemm_lifted_2d / _2d_gather */
} moa_xplan_variant;
#define MOA_XF_GATHER 1       /* C_full given, gathered with NCCL (rows: all-gather / per-rank broadcasts; cols: via workspace) */
#define MOA_XF_FUSED_GATHER 2 /* C_full inside a window: gather fused into the GEMM epilogue, entry/exit barriers */
#define MOA_XF_PULL_B 4       /* rows: B inside a window on every rank: copy-engine pulls of B's k-panels from rank 0 */
#define MOA_XF_DIRECT_B 8     /* rows: every rank's GEMM reads rank 0's B in place over NVLink (moa_gemm_lifted_direct) */
typedef struct {
  int32_t op, comm, root, group, operand, phase, panel, reserved;
  int64_t offset, count;
} moa_coll_t;

/* Fills ops[0..*nops) (at most max_ops; MOA_ERR_INVALID_SHAPE if more are needed,
 * with *nops = the number needed). grid_rows/grid_cols are used by MOA_XPLAN_2D only;
 * npanels as moa_gemm_lifted_ex (0 = static choice). Pure function (no device). */
int moa_exchange_plan(int variant, int64_t m, int64_t n, int64_t p, int dtype, int nranks, int rank, int grid_rows,
                      int grid_cols, int npanels, int flags, moa_coll_t* ops, int max_ops, int* nops);

/* moa_pull_panels — the static k-panel split of B for MOA_XF_PULL_B: the first panel is
 * small (n/64 rows, a multiple of 32, at least 32) so that little of the pull is
 * exposed before the first panel's compute, and each later panel doubles (its pull
 * hides behind the previous panel's compute), at most 16 panels. Writes the panel
 * boundaries bnd[0..K] (bnd[0] = 0, bnd[K] = n) when bnd != NULL; returns K (>= 1). */
int moa_pull_panels(int64_t n, int64_t* bnd);

/* ------------------------------------------------------------------------
 * moa_psi — MoA psi on a row-major array (appendix; bracket bridge
 * rav(i psi xi) == (rav xi)[gamma(i; rho xi)]):
 *   rank, shape[0..rank): rho xi (extents >= 0). rank == 0 is a scalar.
 *   q, idx[0..q): a full (q == rank) or prefix (q < rank) index, 0 <= idx[d] < shape[d].
 *   out: *offset = gamma_row(idx ++ 0...; shape), *count = prod(shape[q..rank)).
 *   psi(idx, xi) is the CONTIGUOUS slice rav(xi)[*offset, *offset + *count).
 * Errors: MOA_ERR_INVALID_INDEX (q > rank, or an index out of bounds),
 * MOA_ERR_INVALID_SHAPE (negative extent or overflow), MOA_ERR_NULL_POINTER.
 * In the ONF, psi(<i>, A) = [i*n, i*n+n) and psi(<sigma>, B) = [sigma*p, sigma*p+p):
 * the contiguous rows of Fig. 1.
 * ------------------------------------------------------------------------ */
int moa_psi(int rank, const int64_t* shape, int q, const int64_t* idx, int64_t* offset, int64_t* count);

/* moa_lift_rows — dimension lifting of the row axis: part `part` of `nparts`
 * (P:142-148). Balanced contiguous split (reading R5; ip_rows.c's sizel/np
 * would drop m mod np rows): rows = floor(m/G) + (g < m mod G),
 * row0 = g*floor(m/G) + min(g, m mod G). Equals the listing's split when G | m.
 * Errors: MOA_ERR_INVALID_SHAPE (m < 0, nparts <= 0, part out of range). */
int moa_lift_rows(int64_t m, int nparts, int part, int64_t* row0, int64_t* rows);

/* moa_plan — the static chooser (no device work; reads cached device props).
 * device < 0 means the current device. */
int moa_plan(int64_t m, int64_t n, int64_t p, int dtype, int device, moa_plan_t* out);

/* moa_select_block_paper — the paper's own block arithmetic: the
 * largest power-of-two side b with three b x b blocks (A, B, C) of
 * elem_bytes each fitting l1_budget_bytes. 32 KiB, 8 -> 32; 128 KiB, 8 -> 64.
 * Errors: MOA_ERR_INVALID_SHAPE if even b = 1 does not fit. */
int moa_select_block_paper(int64_t l1_budget_bytes, int elem_bytes, int64_t* b);

/* ------------------------------------------------------------------------
 * The "ipophp" siblings on the same row-major skeleton (P:372-378, P:515-530:
 * "Matrix Multiplication (MM), Hadamard Product (HP), and the Kronecker Product
 * (KP) using one algorithm/circuit"). dtype MOA_F64 or MOA_F32; device pointers,
 * row-major contiguous; C must not overlap an input; asynchronous on `stream`.
 * One rounding per element, so results equal the oracle bit for bit.
 * moa_hadamard: rho A = rho B = rho C = <m,n>;  C[(i*n)+j] = A[(i*n)+j] * B[(i*n)+j].
 * moa_kron:     A<m,n>, B<p,q>, C<m*p, n*q>;
 *               C[((i*p)+k)*(n*q) + (j*q)+l] = A[(i*n)+j] * B[(k*q)+l]
 *               (the outer product with its middle axes interchanged, ravelled).
 * ------------------------------------------------------------------------ */
int moa_hadamard(int64_t m, int64_t n, const void* A, const void* B, void* C, int dtype, void* stream);
int moa_kron(int64_t m, int64_t n, int64_t p, int64_t q, const void* A, const void* B, void* C, int dtype,
             void* stream);

/* Communicator (library-owned; the 128-byte unique id is shipped by the caller,
 * e.g. over torch.distributed). `device` is the CUDA device the rank uses. */
int moa_comm_get_unique_id(unsigned char id[128]);
int moa_comm_init(int nranks, int rank, const unsigned char id[128], int device, moa_comm_t* comm);
int moa_comm_destroy(moa_comm_t comm);

/* moa_comm_agree — COLLECTIVE, SYNCHRONOUS: *global_status = the maximum over ranks of
 * local_status (e.g. this rank's result of validating its arguments), via a one-int
 * NCCL all-reduce on the communicator's side stream, which this call synchronises.
 * Lets every rank fail together before entering a lifted call. */
int moa_comm_agree(moa_comm_t comm, int local_status, int* global_status);

const char* moa_status_string(int status);
const char* moa_last_error(void);
int moa_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOA_H */
