/*
 * symdiag_b200.h — C ABI of the B200-native batched closed-form 2x2 / 3x3
 * symmetric diagonalizer (arXiv 1306.6291).
 *
 * This is the drop-in boundary: every entry point below replaces one
 * per-matrix function of the reference Python package `symdiag`
 * (/root/reference/pkg/src/symdiag/, cited as file:line) with a batched,
 * stream-ordered launch over caller-owned DEVICE buffers.  No torch types,
 * no allocation on the device entry points, no global mutable state
 * (the only per-thread state is the last error string), reentrant.
 *
 * Packed layouts (row-major upper triangle, AoS):
 *   2x2 : A[n][3] = (a11, a12, a22)                 24 B fp64 per matrix
 *   3x3 : A[n][6] = (a11, a12, a13, a22, a23, a33)  48 B fp64 / 24 B fp32
 * (The reference field orders are SymMat2(a11,a22,a12) core.py:58-60 and
 *  SymMat3(a11,a22,a33,a12,a13,a23) core.py:83-88; the Python layer permutes.)
 *
 * Outputs:
 *   lam[n][3] eigenvalues in SOLVER order (lambda1 >= lambda3 >= lambda2 from
 *             the cosine placement, eig3.py:159-174, or (lam, lam, lam3) on
 *             the double-root branch, eig3.py:492-501, 533-534)
 *   ang[n][3] (phi1, phi2, phi3), each wrapped to (-pi/2, pi/2]
 *             (core.py:115-135).  The Euler angles are the same triple
 *             (eig3.py:568-576), so there is no separate Euler buffer.
 *   status[n] one byte per matrix, see SD_CODE_* / SD_FLAG_* below; rows
 *             whose code is an error (>= SD_ERR_FIRST) carry NaN outputs.
 *
 * Return value of every entry point: SD_OK or an SD_E* launch/argument error
 * (per-matrix outcomes never surface here — they are in `status`).
 */
#ifndef SYMDIAG_B200_H
#define SYMDIAG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define SD_OK 0
#define SD_EINVAL 1      /* bad argument (negative n, null buffer, ...)     */
#define SD_ECUDA 2       /* CUDA launch / runtime error (see sd_last_error) */
#define SD_ENOMEM 3      /* host-plan allocation failed                     */

/* ---- per-matrix status byte -------------------------------------------- */
/* bits 0-3: outcome code.  Branch codes mirror core.Branch (core.py:138-142);
 * error codes mirror the exception taxonomy the reference raises out of
 * diagonalize3.                                       */
#define SD_CODE_MASK 0x0F
#define SD_CODE_GENERIC 0             /* Branch.GENERIC                      */
#define SD_CODE_ALREADY_DIAGONAL_2D 1 /* Branch.ALREADY_DIAGONAL_2D          */
#define SD_CODE_DOUBLE_ROOT 2         /* Branch.DOUBLE_ROOT                  */
#define SD_CODE_TRIPLE_ROOT 3         /* Branch.TRIPLE_ROOT                  */
/* codes 4-7 only appear from the stage-level entry points, for the
 * exceptions diagonalize3 catches and reroutes (eig3.py:547):             */
#define SD_STAGE_DEGENERATE_EIGENVALUES 6 /* DegenerateEigenvalues eig3.py:191-192, 204-205 */
#define SD_STAGE_BOTH_F_ZERO 7            /* BothFVectorsZero      eig3.py:285-286 */
#define SD_ERR_FIRST 8
#define SD_ERR_NONFINITE_INPUT 8      /* NonFiniteInput        core.py:23-26 */
#define SD_ERR_P_NEGATIVE 9           /* ValueError            eig3.py:142-143 */
#define SD_ERR_ACOS_SLACK 10          /* ValueError            eig3.py:153-154 */
#define SD_ERR_DOMAIN_EXCURSION 11    /* DomainExcursion       eig3.py:177-180 via :401 */
#define SD_ERR_NOT_DOUBLE_ROOT 12     /* NotDoubleRoot         eig3.py:397-398 */
#define SD_ERR_ANGLE_OF_ZERO 13       /* AngleOfZeroVector     core.py:241-242 */
#define SD_ERR_MATH_DOMAIN 14         /* ValueError("math domain error") from a math.* call */
#define SD_ERR_OVERFLOW 15            /* OverflowError from float ** (x**n overflow) */
/* bits 4-7: flags */
#define SD_FLAG_S2_NEG 0x10   /* selected sign of phi2 is -1 (post-flip, eig3.py:264-266) */
#define SD_FLAG_S3_NEG 0x20   /* selected sign of phi3 is -1                  */
#define SD_FLAG_NEAR_TIE 0x40 /* SolveReport.near_tie (eig3.py:321, :440)     */
#define SD_FLAG_POLISHED 0x80 /* Gauss-Newton polish accepted (eig3.py:555-561) */

/* ---- report rows (sd_eig3_report_f64) ---------------------------------- */
/* One row of SD_REPORT_STRIDE doubles per matrix, the SolveReport fields
 * (core.py:145-161):
 *   [0] f1_norm  [1] f2_norm  [2] recon_residual  [3] number of candidates
 *   [4 + 5*k + {0..4}] candidate k = (sign2, sign3, phi1_f1g1, phi1_f2g2, diff)
 * Unused candidate slots are NaN.                                          */
#define SD_REPORT_STRIDE 24

/* ---- hot path: full decompositions -------------------------------------- */

/* diagonalize2 (eig2.py:44-48): eigenvalues2 (eig2.py:22-26) + rotation_angle2
 * (eig2.py:29-41).  lam[n][2] = (lambda1, lambda2), phi[n].
 * status: SD_CODE_GENERIC, SD_ERR_NONFINITE_INPUT or SD_ERR_OVERFLOW.      */
int sd_eig2_f64(const double* A, int64_t n, double* lam, double* phi,
                uint8_t* status, void* cuda_stream);

/* diagonalize3 (eig3.py:509-565) in fp64.  Replaces the per-matrix Python
 * loop over diagonalize3 + euler_angles (cli.py:92-95, cli.py:196).        */
int sd_eig3_f64(const double* A, int64_t n, double* lam, double* ang,
                uint8_t* status, void* cuda_stream);

/* diagonalize3 with fp32 input/output and fp64 internal arithmetic.  The
 * reference is fp64-only; inputs are upcast exactly.         */
int sd_eig3_f32(const float* A, int64_t n, float* lam, float* ang,
                uint8_t* status, void* cuda_stream);

/* diagonalize3 plus the SolveReport rows (report[n][SD_REPORT_STRIDE]) and,
 * when d != NULL, the eigenvector matrix D = rot3x.rot3y.rot3z
 * (core.py:229-235) as d[n][9] row-major.  Either of report/d may be NULL. */
int sd_eig3_report_f64(const double* A, int64_t n, double* lam, double* ang,
                       uint8_t* status, double* report, double* d,
                       void* cuda_stream);

/* diagonalize2 plus D = rot2(phi) (core.py:205-208) as d[n][4] row-major.  */
int sd_eig2_report_f64(const double* A, int64_t n, double* lam, double* phi,
                       uint8_t* status, double* d, void* cuda_stream);

/* ---- stage-level entry points (the reference's public stage functions) -- */

/* char_coeffs (eig3.py:102-109): bcd[n][3] = (b, c, d); status: 0,
 * SD_ERR_NONFINITE_INPUT or SD_ERR_OVERFLOW (a**2 overflow, eig3.py:106). */
int sd_char_coeffs_f64(const double* A, int64_t n, double* bcd,
                       uint8_t* status, void* cuda_stream);
/* compute_pq (eig3.py:129-156): pqd[n][3] = (p, q, delta), delta = NaN when
 * the reference returns delta=None (triple root).  status: 0, P_NEGATIVE,
 * ACOS_SLACK, MATH_DOMAIN or OVERFLOW.                                      */
int sd_compute_pq_f64(const double* bcd, int64_t n, double* pqd,
                      uint8_t* status, void* cuda_stream);
/* eigenvalues3 (eig3.py:159-174): lam[n][3] in solver order.               */
int sd_eigenvalues3_f64(const double* bcd, const double* pqd, int64_t n,
                        double* lam, void* cuda_stream);
/* pq_expanded (eig3.py:112-126): pq[n][2]; status as sd_char_coeffs_f64. */
int sd_pq_expanded_f64(const double* A, int64_t n, double* pq,
                       uint8_t* status, void* cuda_stream);
/* compute_v (eig3.py:183-195): v[n]; status: 0,
 * SD_STAGE_DEGENERATE_EIGENVALUES or SD_ERR_DOMAIN_EXCURSION.              */
int sd_compute_v_f64(const double* A, const double* lam, int64_t n,
                     double* v, uint8_t* status, void* cuda_stream);
/* compute_w (eig3.py:198-206) for caller-given v[n]: w[n]; status as above. */
int sd_compute_w_f64(const double* A, const double* lam, const double* v,
                     int64_t n, double* w, uint8_t* status, void* cuda_stream);
/* resolve_signs (eig3.py:269-386) for given lambdas and v, w.  ang[n][3],
 * status carries the sign / near-tie flags; report (nullable) as above.
 * BothFVectorsZero is reported as SD_STAGE_BOTH_F_ZERO.                    */
int sd_resolve_signs_f64(const double* A, const double* lam,
                         const double* vw, int64_t n, double* ang,
                         uint8_t* status, double* report, void* cuda_stream);
/* degenerate_double (eig3.py:389-454): lam2[n][2] = (lam, lam3).          */
int sd_degenerate_double_f64(const double* A, const double* lam2, int64_t n,
                             double* ang, uint8_t* status, double* report,
                             void* cuda_stream);
/* f_vectors (eig3.py:209-213): f[n][4] = (f1x, f1y, f2x, f2y).             */
int sd_f_vectors_f64(const double* A, int64_t n, double* f, void* cuda_stream);
/* g_vectors (eig3.py:216-225): in[n][7] = (l1,l2,l3,phi2,phi3,v,w),
 * g[n][4] = (g1x, g1y, g2x, g2y).                                          */
int sd_g_vectors_f64(const double* in, int64_t n, double* g, void* cuda_stream);
/* compose_rotation (core.py:229-235): ang[n][3] -> d[n][9].                */
int sd_compose_rotation_f64(const double* ang, int64_t n, double* d,
                            void* cuda_stream);

/* ---- independent referees (SURVEY §8f "next" rows) ---------------------- */

/* jacobi_eigen (oracle.py:45-84): cyclic-by-row Jacobi on packed rows of
 * dimension dim (2: (a11,a12,a22); 3: six values) until the off-diagonal
 * mass is <= tol^2 max(1, ||A||_F^2).  evals[n][dim] (final diagonal),
 * evecs[n][dim*dim] row-major (columns are eigenvectors), sweeps[n],
 * offdiag[n] (sqrt of the final off-diagonal sum of squares).
 * status: 0, 1 = NoConvergence (oracle.py:63-64, > 100 sweeps),
 * SD_ERR_NONFINITE_INPUT.                                                  */
int sd_jacobi_f64(int dim, const double* A, int64_t n, double tol, double* evals,
                  double* evecs, int32_t* sweeps, double* offdiag, uint8_t* status,
                  void* cuda_stream);
/* residuals (oracle.py:144-161) of a decomposition (lam[n][dim], d[n][dim*dim]
 * row-major): out[n][dim+2] = (recon_rel, ortho, eigvec_res[0..dim-1]).    */
int sd_residuals_f64(int dim, const double* A, const double* lam, const double* d,
                     int64_t n, double* out, void* cuda_stream);

/* cubic_roots_reference (oracle.py:87-133): bcd[n][3] = (b, c, d) of
 * l^3 - b l^2 + c l + d -> roots[n][3] (ascending brackets, repeated roots
 * as the reference orders them); status 0 or 1 = ComplexRootsDetected.    */
int sd_cubic_roots_f64(const double* bcd, int64_t n, double* roots,
                       uint8_t* status, void* cuda_stream);

/* x[i] ** y[i] with the reference's pow: CPython float ** float is libm
 * pow, i.e. glibc 2.39's pow (e_pow.c, the FMA build on x86-64), restated
 * bit for bit for the device (csrc/sd_glibc_pow.h); y integer-valued with
 * 2^-65 <= |y| < 2^63 (the reference raises to 2, 3 and 6).  Replaces the
 * `**` of eig3.py:89, 99, 105-108, 140, 147, 151 and core.py:107-108.     */
int sd_glibc_pow_f64(const double* x, const double* y, int64_t n, double* out,
                     void* cuda_stream);

/* The literal solver's libm, elementwise: fn 0 sin(x), 1 cos(x), 2 acos(x),
 * 3 asin(x), 4 atan2(x, y), 5 hypot(x, y) (y may be NULL for fn < 4),
 * correctly rounded (csrc/sd_crlibm.h: a quick double-double phase with a
 * rounding test, an accurate phase behind it), i.e. the value CPython's
 * math.sin / cos / acos / asin / atan2 / hypot return on the reference's
 * host wherever glibc itself rounds correctly.  Replaces the libm calls of
 * eig3.py:143-174, 218-246, 288-379 and core.py:238-246 on the rows the
 * literal pass solves.                                                       */
int sd_crlibm_f64(int fn, const double* x, const double* y, int64_t n, double* out,
                  void* cuda_stream);

/* ---- host-buffer path (end-to-end: H2D, kernel, D2H, pipelined) ---------- */
typedef struct sd_plan sd_plan;
/* A plan owns three device staging slots of `chunk` matrices and three CUDA
 * streams on `device` (copy-in / compute / copy-out of neighbouring chunks
 * overlap).                                                                 */
int sd_plan_create(int device, int64_t chunk, sd_plan** out);
int sd_plan_destroy(sd_plan* plan);
/* Host-memory variants of sd_eig3_f64 / sd_eig3_f32 / sd_eig2_f64.  Copies
 * chunk i+1 in while chunk i computes and chunk i-1 copies out; returns when
 * all outputs are in host memory.  Pinned host memory gives full overlap.  */
int sd_eig3_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam,
                     double* ang, uint8_t* status);
int sd_eig3_f32_host(sd_plan* plan, const float* A, int64_t n, float* lam,
                     float* ang, uint8_t* status);
int sd_eig2_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam,
                     double* phi, uint8_t* status);
/* Synchronous host-buffer sd_eig3_report_f64 / sd_eig2_report_f64 (report /
 * d may be NULL): the low-latency path of the reference-style scalar calls
 * (diagonalize3(SymMat3), diagonalize2(SymMat2)).  Host buffers may be
 * pageable.                                                                 */
int sd_eig3_report_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam,
                            double* ang, uint8_t* status, double* report, double* d);
int sd_eig2_report_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam,
                            double* phi, uint8_t* status, double* d);

/* ---- JSON-lines codec of the `solve` front end (host only, no CUDA) -------
 * Replaces the per-record json.loads / dumps of the reference CLI
 * (cli.py:51-80 parse_record, cli.py:33-48 + 83-114 result records).      */
/* Split buf[0, len) into lines, drop blank ones (str.strip semantics for
 * ASCII) and parse up to `cap` of them with `nthreads` host threads.  Per
 * line k: kind[k] = 3 or 2 with rows[6k ..] = packed (a11,a12,a13,a22,a23,a33)
 * or (a11,a12,a22); or 0 when the line is not a record this parser can read
 * exactly like json.loads + parse_record (malformed, non-finite, non-numeric,
 * duplicate or unexpected keys, escaped / non-ASCII id, ...): the caller
 * parses it.  span[4k ..] = line begin, end, id token begin, end (-1: id
 * absent or null); offsets into buf.  Returns the line count (< 0 on bad
 * arguments); *consumed = bytes of buf covered by those lines.              */
int64_t sd_jsonl_parse(const char* buf, int64_t len, int64_t cap, int nthreads,
                       int8_t* kind, double* rows, int64_t* span, int64_t* consumed);
/* Format ResultRecords (one per line, '\n'-terminated) for records k with
 * dim[k] in {2, 3}; dim[k] = 0 skips k (offsets[k] == offsets[k+1]).  Per
 * record: id token idbuf[id_span[2k], id_span[2k+1]) or null, lam[3k ..],
 * ang[3k ..] (2x2: phi at ang[3k]), d[9k ..] row-major D (2x2: 4 values),
 * res[5k ..] = (recon_rel, ortho, eigvec residuals), status[k] (branch).
 * Returns the byte count written to out, -(needed) if out_cap is too small,
 * or -1 on bad arguments; offsets[n+1] receives record boundaries.         */
int64_t sd_jsonl_format(int64_t n, const int8_t* dim, const char* idbuf,
                        const int64_t* id_span, const double* lam, const double* ang,
                        const double* d, const double* res, const uint8_t* status,
                        int nthreads, char* out, int64_t out_cap, int64_t* offsets);

/* ---- diagnostics --------------------------------------------------------- */
/* sd_eig3_f64 evaluated entirely in the reference's literal evaluation
 * order (one thread per row, no fast path, no deferral).  Same outputs up
 * to the parity tolerance; used to cross-check the fast path.             */
int sd_eig3_literal_f64(const double* A, int64_t n, double* lam, double* ang,
                        uint8_t* status, void* cuda_stream);
/* Only the first (fast, classifying) pass of sd_eig3_f64: rows it could not
 * finish keep internal codes 4 (deferred to the literal solver; bits 4-7 =
 * reason, see sd_fast3.cuh) or 5-7 (closed form written, polish pending).
 * Diagnostics: measures how much of a workload takes the fast path.        */
int sd_eig3_classify_f64(const double* A, int64_t n, double* lam, double* ang,
                         uint8_t* status, void* cuda_stream);
/* FP64-pipe peak probe for the roofline denominator: `blocks` x 256 threads,
 * each runs `iters` x 16 independent DFMA chains; *dfma_total receives the
 * DFMA count (time it with events on `cuda_stream`).  sink[blocks*256].     */
int sd_probe_dfma(int blocks, int iters, double* sink, double* dfma_total,
                  void* cuda_stream);

/* ---- misc --------------------------------------------------------------- */
const char* sd_last_error(void);   /* thread-local message of the last error */
const char* sd_version(void);
/* Number of kernel launches this thread has issued through the library.    */
int64_t sd_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SYMDIAG_B200_H */
