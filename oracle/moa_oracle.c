/* oracle/moa_oracle.c — CPU ORACLE for the MoA-ONF GEMM.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product
 * (paper_2306_11148_b200/) never links, imports or calls it, and shares no code
 * with it (not even headers).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   Eq. 3, the MoA Operational Normal Form of GEMM:
 *       C[(i*p)+j] := sum_{k=0}^{n-1} A[(i*n)+k] * B[(k*p)+j]
 *   over row-major contiguous A<m,n>, B<n,p>, C<m,p> (Eq. 1; index
 *   bounds Eq. 2).
 *
 * How: each routine is a listing of the paper written out literally, in the
 * paper's loop order and index expressions, with the paper's variable names
 * (sizel = m, sizer = p, shr0 = n; `sizeres` and `np` are unused by ip.c).
 *   - oracle_ip_*        : Fig. 3 ip.c, loop order i-sigma-j.
 *   - oracle_ip_rows_*   : Fig. 4 ip_rows.c, row lifting
 *                          i = ip + (sizel/np)*k; k = processor index, run as one
 *                          thread per k (the all-core CPU baseline).
 *   - oracle_ip_cols_*   : Fig. 5 ip_cols.c, j = jp*rsize + kp.
 *   - oracle_ip_ijk_*    : the classical row-times-column definition the paper
 *                          contrasts against ("a row of A with a column
 *                          of B"); brute force used to cross-check ip.c.
 * Readings:
 *   R1  Eq. 3 says ":=" but ip.c accumulates C = C + ...: every routine first
 *       sets C := +0 and then runs the listing (overwrite semantics).
 *   R3  The paper never says whether `C + A*B` is contracted to a fused
 *       multiply-add. Both variants are provided: *_unfused (two roundings,
 *       compiled with -ffp-contract=off) and *_fma (C99 fma(), one rounding per
 *       step — what an FMA-contracting compiler such as the OpenACC toolchain
 *       the paper used emits for this statement). Summation order is the
 *       listing's: sigma ascending.
 *   R5  ip_rows.c / ip_cols.c assume exact division (sizel/np, sizer/rsize);
 *       these literal routines reject non-dividing arguments (return -1)
 *       instead of silently dropping rows.
 * Element types: double (the paper's) and float (north_star extension).
 * Pins: tests/test_oracle.py (exact rational arithmetic within the Higham
 * bound, exact-fma brute force, integer exactness, identities, closed forms,
 * worked examples in tests/golden/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* ---------------- Fig. 3: ip.c ---------------- */
#define DEF_IP(NAME, T, UPDATE)                                                   \
  void NAME(T* C, const T* A, const T* B, i64 sizel, i64 sizer, i64 shr0) {       \
    i64 i, j, sigma;                                                              \
    for (i = 0; i < sizel * sizer; i++) C[i] = (T)0; /* R1: C := 0 first */       \
    for (i = 0; i < sizel; i++) {                                                 \
      for (sigma = 0; sigma < shr0; sigma++) {                                    \
        for (j = 0; j < sizer; j++) {                                             \
          UPDATE(C[j + i * sizer], A[(i * shr0) + sigma], B[(sigma * sizer) + j]); \
        }                                                                         \
      }                                                                           \
    }                                                                             \
  }

#define UPD_UNFUSED(c, a, b) (c) = (c) + (a) * (b)
#define UPD_FMA64(c, a, b) (c) = fma((a), (b), (c))
#define UPD_FMA32(c, a, b) (c) = fmaf((a), (b), (c))

DEF_IP(oracle_ip_unfused_f64, double, UPD_UNFUSED)
DEF_IP(oracle_ip_fma_f64, double, UPD_FMA64)
DEF_IP(oracle_ip_unfused_f32, float, UPD_UNFUSED)
DEF_IP(oracle_ip_fma_f32, float, UPD_FMA32)

/* ---- ip.c restricted to a set of rows (Fig. 1: rows of C are independent).
 * Cout is nrows x sizer: Cout[r*sizer + j] = row rows[r] of ip.c's C. The loop
 * body is ip.c's with i = rows[r]. Returns -1 on an out-of-range row. */
#define DEF_IP_ROWSET(NAME, T, UPDATE)                                            \
  int NAME(T* Cout, const T* A, const T* B, i64 sizel, i64 sizer, i64 shr0,       \
           const i64* rows, i64 nrows) {                                          \
    i64 r, j, sigma;                                                              \
    for (r = 0; r < nrows; r++)                                                   \
      if (rows[r] < 0 || rows[r] >= sizel) return -1;                             \
    for (r = 0; r < nrows * sizer; r++) Cout[r] = (T)0;                           \
    for (r = 0; r < nrows; r++) {                                                 \
      i64 i = rows[r];                                                            \
      for (sigma = 0; sigma < shr0; sigma++) {                                    \
        for (j = 0; j < sizer; j++) {                                             \
          UPDATE(Cout[j + r * sizer], A[(i * shr0) + sigma], B[(sigma * sizer) + j]); \
        }                                                                         \
      }                                                                           \
    }                                                                             \
    return 0;                                                                     \
  }

DEF_IP_ROWSET(oracle_ip_rowset_unfused_f64, double, UPD_UNFUSED)
DEF_IP_ROWSET(oracle_ip_rowset_fma_f64, double, UPD_FMA64)
DEF_IP_ROWSET(oracle_ip_rowset_unfused_f32, float, UPD_UNFUSED)
DEF_IP_ROWSET(oracle_ip_rowset_fma_f32, float, UPD_FMA32)

/* ---- Same, but A is given as only the selected rows (Arows is nrows x shr0), so a
 * caller holding a row sample of a huge A need not materialise all of it. */
#define DEF_IP_ROWBLOCK(NAME, T, UPDATE)                                          \
  void NAME(T* Cout, const T* Arows, const T* B, i64 nrows, i64 sizer, i64 shr0) { \
    i64 r, j, sigma;                                                              \
    for (r = 0; r < nrows * sizer; r++) Cout[r] = (T)0;                           \
    for (r = 0; r < nrows; r++)                                                   \
      for (sigma = 0; sigma < shr0; sigma++)                                      \
        for (j = 0; j < sizer; j++)                                               \
          UPDATE(Cout[j + r * sizer], Arows[(r * shr0) + sigma], B[(sigma * sizer) + j]); \
  }
DEF_IP_ROWBLOCK(oracle_ip_rowblock_unfused_f64, double, UPD_UNFUSED)
DEF_IP_ROWBLOCK(oracle_ip_rowblock_fma_f64, double, UPD_FMA64)
DEF_IP_ROWBLOCK(oracle_ip_rowblock_unfused_f32, float, UPD_UNFUSED)
DEF_IP_ROWBLOCK(oracle_ip_rowblock_fma_f32, float, UPD_FMA32)

/* ---------------- Fig. 4: ip_rows.c ----------------
 * The k loop ("assigns an index to processors") runs one pthread per
 * k; each thread executes the listing's ip/sigma/j loops for its k. */
typedef struct {
  void* C; const void* A; const void* B;
  i64 sizel, sizer, np, shr0, k;
  int fused;
} rows_arg;

static void* ip_rows_worker_f64(void* vp) {
  rows_arg* a = (rows_arg*)vp;
  double* C = (double*)a->C; const double* A = (const double*)a->A; const double* B = (const double*)a->B;
  i64 sizel = a->sizel, sizer = a->sizer, np = a->np, shr0 = a->shr0, k = a->k, ip, sigma, j;
  for (ip = 0; ip < (sizel / np); ip++)
    for (sigma = 0; sigma < shr0; sigma++)
      for (j = 0; j < sizer; j++) {
        if (a->fused)
          UPD_FMA64(C[j + (ip + (sizel / np) * k) * sizer], A[((ip + ((sizel / np) * k)) * shr0) + sigma],
                    B[(sigma * sizer) + j]);
        else
          UPD_UNFUSED(C[j + (ip + (sizel / np) * k) * sizer], A[((ip + ((sizel / np) * k)) * shr0) + sigma],
                      B[(sigma * sizer) + j]);
      }
  return NULL;
}

static void* ip_rows_worker_f32(void* vp) {
  rows_arg* a = (rows_arg*)vp;
  float* C = (float*)a->C; const float* A = (const float*)a->A; const float* B = (const float*)a->B;
  i64 sizel = a->sizel, sizer = a->sizer, np = a->np, shr0 = a->shr0, k = a->k, ip, sigma, j;
  for (ip = 0; ip < (sizel / np); ip++)
    for (sigma = 0; sigma < shr0; sigma++)
      for (j = 0; j < sizer; j++) {
        if (a->fused)
          UPD_FMA32(C[j + (ip + (sizel / np) * k) * sizer], A[((ip + ((sizel / np) * k)) * shr0) + sigma],
                    B[(sigma * sizer) + j]);
        else
          UPD_UNFUSED(C[j + (ip + (sizel / np) * k) * sizer], A[((ip + ((sizel / np) * k)) * shr0) + sigma],
                      B[(sigma * sizer) + j]);
      }
  return NULL;
}

/* elem = 8 (double) or 4 (float). Returns 0, or -1 if np does not divide sizel (R5). */
int oracle_ip_rows(void* C, const void* A, const void* B, i64 sizel, i64 sizer, i64 np, i64 shr0, int elem,
                   int fused) {
  i64 k, i;
  if (np <= 0 || sizel % np != 0 || (elem != 8 && elem != 4)) return -1;
  if (elem == 8) for (i = 0; i < sizel * sizer; i++) ((double*)C)[i] = 0.0;
  else for (i = 0; i < sizel * sizer; i++) ((float*)C)[i] = 0.0f;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)np);
  rows_arg* args = (rows_arg*)malloc(sizeof(rows_arg) * (size_t)np);
  if (!th || !args) { free(th); free(args); return -2; }
  for (k = 0; k < np; k++) {
    rows_arg t = {C, A, B, sizel, sizer, np, shr0, k, fused};
    args[k] = t;
    pthread_create(&th[k], NULL, elem == 8 ? ip_rows_worker_f64 : ip_rows_worker_f32, &args[k]);
  }
  for (k = 0; k < np; k++) pthread_join(th[k], NULL);
  free(th); free(args);
  return 0;
}

/* ---------------- Fig. 5: ip_cols.c, double, unfused ---------------- */
int oracle_ip_cols_unfused_f64(double* C, const double* A, const double* B, i64 sizel, i64 sizer, i64 shr0,
                               i64 rsize) {
  i64 i, jp, kp, sigma;
  if (rsize <= 0 || sizer % rsize != 0) return -1;
  for (i = 0; i < sizel * sizer; i++) C[i] = 0.0;
  for (i = 0; i < sizel; i++)
    for (sigma = 0; sigma < shr0; sigma++)
      for (jp = 0; jp < (sizer / rsize); jp++)
        for (kp = 0; kp < rsize; kp++)
          C[((jp * rsize) + kp) + i * sizer] =
              C[((jp * rsize) + kp) + i * sizer] + A[(i * shr0) + sigma] * B[(sigma * sizer) + ((jp * rsize) + kp)];
  return 0;
}

/* ------- classical row-times-column brute force (SPEC gemm_naive S:205-213) ------- */
void oracle_ip_ijk_unfused_f64(double* C, const double* A, const double* B, i64 m, i64 p, i64 n) {
  for (i64 i = 0; i < m; i++)
    for (i64 j = 0; j < p; j++) {
      double s = 0.0;
      for (i64 k = 0; k < n; k++) s = s + A[i * n + k] * B[k * p + j];
      C[i * p + j] = s;
    }
}
void oracle_ip_ijk_unfused_f32(float* C, const float* A, const float* B, i64 m, i64 p, i64 n) {
  for (i64 i = 0; i < m; i++)
    for (i64 j = 0; j < p; j++) {
      float s = 0.0f;
      for (i64 k = 0; k < n; k++) s = s + A[i * n + k] * B[k * p + j];
      C[i * p + j] = s;
    }
}

/* fp32 inputs, fp64 accumulation, single final rounding per element: the
 * reference "truth" used only to REPORT the error of the TF32 variant
 * (north_star: "TF32 variant <= 5e-3, reported separately"). */
void oracle_ip_f32_in_f64_acc(double* C, const float* A, const float* B, i64 sizel, i64 sizer, i64 shr0) {
  for (i64 i = 0; i < sizel * sizer; i++) C[i] = 0.0;
  for (i64 i = 0; i < sizel; i++)
    for (i64 sigma = 0; sigma < shr0; sigma++)
      for (i64 j = 0; j < sizer; j++)
        C[j + i * sizer] = C[j + i * sizer] + (double)A[(i * shr0) + sigma] * (double)B[(sigma * sizer) + j];
}

/* ---------------- ipophp siblings ----------------
 * "scalar operations: Matrix Multiplication (MM), Hadamard Product (HP), and the
 * Kronecker Product (KP) using one algorithm/circuit (ipophp)".
 * Hadamard: rho A = rho B = <m,n>; C[(i*n)+j] = A[(i*n)+j] * B[(i*n)+j]
 *   (pointwise scalar operation; indexing distributes over it).
 * Kronecker: A<m,n>, B<p,q> -> C<m*p, n*q>, the outer product (rank 4,
 *   <m,n,p,q>) with its two middle axes interchanged and ravelled row-major:
 *   C[((i*p)+k)*(n*q) + (j*q)+l] = A[(i*n)+j] * B[(k*q)+l].
 * One rounding per element (a single product): exact results are unique. */
void oracle_hadamard_f64(double* C, const double* A, const double* B, i64 m, i64 n) {
  for (i64 i = 0; i < m; i++)
    for (i64 j = 0; j < n; j++) C[(i * n) + j] = A[(i * n) + j] * B[(i * n) + j];
}
void oracle_hadamard_f32(float* C, const float* A, const float* B, i64 m, i64 n) {
  for (i64 i = 0; i < m; i++)
    for (i64 j = 0; j < n; j++) C[(i * n) + j] = A[(i * n) + j] * B[(i * n) + j];
}
void oracle_kron_f64(double* C, const double* A, const double* B, i64 m, i64 n, i64 p, i64 q) {
  for (i64 i = 0; i < m; i++)
    for (i64 j = 0; j < n; j++)
      for (i64 k = 0; k < p; k++)
        for (i64 l = 0; l < q; l++) C[((i * p) + k) * (n * q) + (j * q) + l] = A[(i * n) + j] * B[(k * q) + l];
}
void oracle_kron_f32(float* C, const float* A, const float* B, i64 m, i64 n, i64 p, i64 q) {
  for (i64 i = 0; i < m; i++)
    for (i64 j = 0; j < n; j++)
      for (i64 k = 0; k < p; k++)
        for (i64 l = 0; l < q; l++) C[((i * p) + k) * (n * q) + (j * q) + l] = A[(i * n) + j] * B[(k * q) + l];
}
