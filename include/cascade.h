/*
 * cascade.h -- C ABI of the B200 (sm_100a) fast-cascade library  libcascade_b200.so
 *
 * Implements the time-domain cascade of G. Beylkin, "Fast convolution algorithm for state
 * space models", arXiv 2411.17729 (PAPER.md in the reference tree; line numbers below).
 *
 *   Problem (§3): given the discrete LTI system of Eq. 2,
 *     x_l = Abar x_{l-1} + Bbar u_l,   y_l = C x_l + D u_l,   x_{-1} = 0,
 *   produce {y_l}_{l=0}^{L-1} for the truncated transfer function H_N of Eq. 5
 *   (PAPER.md:132-135):  H_N(z) = C prod_{n=0}^{N} [I + (z^-1 Abar)^(2^n)] Bbar + D.
 *   Method: v^(0)_l = Bbar u_l; for k = 0..N (N+1 stages, R1),
 *     v_l <- v_l + Abar^(2^k) v_{l-2^k}  for l >= 2^k (out of place; l < 2^k unchanged);
 *     y_l = C v_l + D u_l.
 *   The powers Abar^(2^k) come from repeated squaring.
 *
 * Conventions for every entry point
 *   - Plain pointers and sizes only; no torch or CUDA types. `stream` is a cudaStream_t
 *     passed as void* (NULL = legacy default stream).
 *   - Ownership: the caller allocates every buffer (device memory unless stated) including
 *     the workspace, sized by the matching *_bytes query. The library never allocates or
 *     frees device memory inside an apply call and keeps no state between calls
 *     (stateless; thread-safe for distinct workspaces). casc_run_host calls on one device are
 *     serialised by the library (they share its per-device copy streams and pinned staging).
 *   - Asynchrony: all device work is enqueued on `stream`; no host synchronisation inside
 *     casc_powers / casc_apply / casc_apply_bank. casc_run_host synchronises `stream` once
 *     at its end (its output lives in host memory).
 *   - Errors: returned as casc_status; nothing is thrown across the ABI. Arguments are
 *     validated before any work is enqueued. There is NO CPU fallback: a shape or mode the
 *     GPU kernels do not cover returns CASC_ERR_UNSUPPORTED.
 *   - Empty calls: casc_powers with n_sys = 0, and casc_apply / casc_apply_bank /
 *     casc_run_host with n = 0, L = 0 or batch = 0 (the other sizes and the mode still
 *     valid) return CASC_OK without touching any buffer (pointers may be NULL; the *_bytes
 *     queries return 0). casc_apply_seqsharded requires L_loc >= 1 and batch >= 1.
 *   - Precision modes: CASC_FP32 stores signals and states in fp32 and computes with fp32
 *     accuracy (two-part operand splits with 22 significant bits: 3xTF32 tensor-core products,
 *     or, in the m = 64 bank head, the same three products of fp16 parts under exact
 *     power-of-two scales (R33); fp32 accumulation; tolerance 1e-5 relative L2,
 *     BASELINE north_star); CASC_BF16 stores signals/states in bf16 and accumulates in fp32
 *     (tolerance 2e-2). Model parameters (Abar, Bbar, C, D) are always passed in float64 and
 *     rounded once, inside the library, to the format the kernels consume.
 *   - Layouts (row-major, C order): Abar [n_sys][m][m]; Bbar [n_sys][m][p]; C [n_sys][q][m];
 *     D [n_sys][q][p] (may be NULL = 0); u [n_sys][batch][L][p]; y [n_sys][batch][L][q].
 *     Time is the second-fastest axis of a signal; the shift by 2^k stays inside one
 *     sequence (one (system, batch) pair) and reads zeros before l = 0.
 */
#ifndef CASCADE_B200_H
#define CASCADE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum casc_status {
  CASC_OK = 0,
  CASC_ERR_ARG = 1,          /* null pointer, m/p/q < 1, L/batch < 0, N < 0, bad mode       */
  CASC_ERR_DIM = 2,          /* inconsistent dimensions (e.g. p > m, N > N_max)               */
  CASC_ERR_NONSQUARE = 3,    /* reserved: Abar is square by construction of the ABI          */
  CASC_ERR_UNSUPPORTED = 4,  /* valid request the sm_100a kernels do not cover                */
  CASC_ERR_WORKSPACE = 5,    /* ws_bytes smaller than the *_bytes query                       */
  CASC_ERR_CUDA = 6,         /* a CUDA runtime call failed (launch, copy, device mismatch)    */
  CASC_ERR_NCCL = 7          /* NCCL missing or an NCCL call failed (sequence-sharded path)   */
} casc_status;

typedef enum casc_mode {
  CASC_FP32 = 0,             /* fp32 storage, fp32-accurate math (split-operand tensor cores) */
  CASC_BF16 = 1              /* bf16 storage, fp32 accumulation                               */
} casc_mode;

/* Human-readable name of a status code (static string). */
const char* casc_status_str(int status);

/* Library version (major*10000 + minor*100 + patch) and the compute capability it targets
 * (100 = sm_100a). */
int casc_version(void);
int casc_target_sm(void);

/* ----------------------------------------------------------------------------------------
 * a1  Powers by repeated squaring -- PAPER.md:164-166 ("we need to compute the powers of
 *     the matrix Abar, Abar^2, Abar^4, Abar^8, ..."); accuracy remark PAPER.md:274-277.
 *
 * For each system s: P_0 = Abar_s, P_{k+1} = P_k P_k (float64 throughout, k < N_s), then
 * each P_k (k <= N_s) is rounded once to the storage format of `mode` (fp32: tf32 hi + tf32
 * lo pair, round-to-nearest-away; bf16: round-to-nearest-even).
 *   n_sys   number of independent systems (1 for a single MIMO system).
 *   m       state dimension (Abar is m x m).
 *   N_host  HOST int array [n_sys]: truncation order N_s (0 <= N_s <= N_max).
 *   N_max   slot count of the pack (pack holds N_max+1 powers per system).
 *   Abar    DEVICE float64 [n_sys][m][m], read only.
 *   pack    DEVICE buffer of casc_pack_bytes(n_sys, m, N_max, mode) bytes, written. Opaque:
 *           consumed only by casc_apply / casc_apply_bank with the same (n_sys, m, N_max, mode).
 * Errors: CASC_ERR_ARG (null, m < 1, n_sys < 1, N_max < 0), CASC_ERR_DIM (N_s out of range),
 *         CASC_ERR_UNSUPPORTED (m > 4096), CASC_ERR_CUDA.
 * -------------------------------------------------------------------------------------- */
size_t casc_pack_bytes(int n_sys, int m, int N_max, int mode);
int casc_powers(int n_sys, int m, const int* N_host, int N_max, const double* Abar, int mode,
                void* pack, void* stream);
/* a0 / a1 diagnostics for the planner (SURVEY §8(b) tail_norm_fro): the Frobenius norms of the
 * float64 powers in `pack`, ||P_k||_F for k = 0..N_s, and of the first neglected power
 * ||P_{N_s+1}||_F = ||P_{N_s} P_{N_s}||_F, whose size sets the truncation error of H_N
 * (the error term is (z^-1 Abar)^(2^(N+1)) times a bounded factor). P_{N_s+1}
 * is formed block by block in float64 and reduced, never stored.
 *   pack        DEVICE, from casc_powers(n_sys, m, N_host, N_max, mode, ...).
 *   norms_host  HOST double [n_sys][N_max + 2] (written): entry k of system s; NaN for k > N_s + 1.
 * Synchronises `stream` (host output). Errors: CASC_ERR_ARG, CASC_ERR_DIM, CASC_ERR_CUDA. */
int casc_powers_norms(int n_sys, int m, int N_max, int mode, const void* pack, double* norms_host, void* stream);

/* ----------------------------------------------------------------------------------------
 * a2-a5  Apply one LTI system (MIMO or SISO) to `batch` sequences of length L --
 *     PAPER.md:185-229 (§3): v^(0) = Bbar u (:187), N+1 out-of-place shifted stages
 *     (:193-225, general step :217-225), y = C v + D u (:226-229). Stages with 2^k >= L are
 *     the identity and are skipped (R20).
 *   m, p, q   state / input / output dimensions (1 <= p, q <= m).
 *   L, batch  sequence length and number of sequences.
 *   N         truncation order (N+1 stages); pack must come from casc_powers with N_s = N.
 *   mode      CASC_FP32 (u, y are float32) or CASC_BF16 (u, y are bf16 bit patterns).
 *   pack      DEVICE, from casc_powers(1, m, &N, N_max, ...) (N_max is read from the call
 *             that built it: pass it again as N_max).
 *   Bbar, C, D  DEVICE float64 [m][p], [q][m], [q][p] (D may be NULL meaning D = 0).
 *   u         DEVICE [batch][L][p];  y  DEVICE [batch][L][q] (written).
 *   ws        DEVICE workspace of >= casc_apply_workspace_bytes(...) bytes.
 *   effective_stages  HOST int* (may be NULL): #{k <= N : 2^k < L}.
 * Errors: CASC_ERR_ARG, CASC_ERR_DIM (p > m or q > m), CASC_ERR_WORKSPACE,
 *         CASC_ERR_UNSUPPORTED, CASC_ERR_CUDA.
 * -------------------------------------------------------------------------------------- */
size_t casc_apply_workspace_bytes(int m, int p, int q, int64_t L, int batch, int N, int mode);
int casc_apply(int m, int p, int q, int64_t L, int batch, int N, int N_max, int mode,
               const void* pack, const double* Bbar, const double* C, const double* D,
               const void* u, void* y, void* ws, size_t ws_bytes, int* effective_stages,
               void* stream);

/* ----------------------------------------------------------------------------------------
 * a6  Bank of independent SISO channels (p = q = 1), each with its own (Abar_c, Bbar_c,
 *     C_c, D_c, N_c) -- the HiPPO example of PAPER.md:253-273 (Eq. 9-10) applied per
 *     channel with the cascade of PAPER.md:185-229.
 *   n_ch      number of channels; N_host HOST int [n_ch]; pack from
 *             casc_powers(n_ch, m, N_host, N_max, ...).
 *   Bbar      DEVICE float64 [n_ch][m]; C DEVICE float64 [n_ch][m]; D DEVICE float64 [n_ch]
 *             (may be NULL = 0).
 *   u, y      DEVICE [n_ch][batch][L] in the storage dtype of `mode`.
 *   ws_bytes  may be smaller than casc_bank_workspace_bytes(n_ch, ...): the channels are then
 *             processed in consecutive waves of as many channels as fit (bounded memory, e.g.
 *             BASELINE configs[4]: 4096 x 8 x 65536 x 64 fp32 states = 550 GB per buffer); at
 *             least casc_bank_workspace_bytes(1, ...) is required.
 * Errors as casc_apply.
 * -------------------------------------------------------------------------------------- */
size_t casc_bank_workspace_bytes(int n_ch, int m, int64_t L, int batch, int N_max, int mode);
int casc_apply_bank(int n_ch, int m, int64_t L, int batch, const int* N_host, int N_max,
                    int mode, const void* pack, const double* Bbar, const double* C,
                    const double* D, const void* u, void* y, void* ws, size_t ws_bytes,
                    void* stream);

/* ----------------------------------------------------------------------------------------
 * End-to-end entry with HOST buffers: copies Abar, Bbar, C, D (float64) and u (storage
 * dtype) host -> device, runs casc_powers + casc_apply / casc_apply_bank, copies y back to
 * host, and synchronises `stream`. Host buffers should be pinned for asynchronous copies.
 *   n_sys == 1 with any (p, q) runs the single-system path; n_sys > 1 requires p = q = 1
 *   (bank). dev_ws: DEVICE buffer of casc_run_host_bytes(...) bytes; for banks a smaller
 *   buffer is accepted (its tail becomes the apply workspace and the channels run in waves).
 * -------------------------------------------------------------------------------------- */
size_t casc_run_host_bytes(int n_sys, int m, int p, int q, int64_t L, int batch, int N_max,
                           int mode);
int casc_run_host(int n_sys, int m, int p, int q, int64_t L, int batch, const int* N_host,
                  int N_max, int mode, const double* Abar_h, const double* Bbar_h,
                  const double* C_h, const double* D_h, const void* u_h, void* y_h,
                  void* dev_ws, size_t dev_ws_bytes, void* stream);

/* ----------------------------------------------------------------------------------------
 * a7  Sequence-sharded apply (BASELINE configs[3] "per-stage NCCL halo exchange").
 *     Rank r of `world` owns global time rows [r*L_loc, (r+1)*L_loc) of every sequence of ONE
 *     system (m, p, q multiples of 64). The cascade's stage k reads
 *     v_{l-2^k}, so before stage k each rank receives the last 2^k time rows of v^(k) from rank
 *     r-1 (zeros on rank 0: x_{-1} = 0); the first step needs 3 rows of u (the
 *     Krylov head over four lags, R28; 1 row when Ne = 1), the output step the rows of v
 *     it reads before l: 2^Ne of v^(Ne) (y = C v + C P_Ne v_{l-2^Ne} + D u, R21) or, for Ne >= 3,
 *     3 * 2^(Ne-1) of v^(Ne-1) (the last stage folded into y, R31).
 *     Ne = min(N, floor(log2(L - 1))) for the GLOBAL length L = world * L_loc (R20).
 *     The library does the exchange itself: grouped ncclSend(r -> r+1) / ncclRecv(r-1 -> r) on
 *     `comm_stream`, overlapped with the interior rows of the same step on `compute_stream`
 *     (rows whose operands are all local run first; the boundary rows after the halo landed).
 *
 *   casc_nccl_unique_id  writes the 128-byte NCCL unique id (call on rank 0; the caller
 *                        broadcasts it, e.g. through its torch process group).
 *   casc_comm_init       NCCL communicator of `world` ranks on the CURRENT device (the caller has
 *                        done cudaSetDevice(local_rank)); blocks until every rank joined.
 *   casc_comm_init_local `world` emulated ranks in ONE process on one device (tests: comms[r]
 *                        is rank r; each rank's apply must run on its own host thread; halos are
 *                        device copies ordered by events).
 *   casc_comm_destroy    frees a communicator from either init.
 *   casc_comm_rank       rank and world size of a communicator (either pointer may be NULL).
 *
 *   Layouts (time-major, so a halo of d rows is ONE contiguous block of d*batch*dim elements):
 *     u_loc DEVICE [L_loc][batch][p], y_loc DEVICE [L_loc][batch][q] (storage dtype of mode);
 *     pack from casc_powers(1, m, &N, N_max, ...); Bbar, C, D float64 as casc_apply (D may be NULL).
 *     ws: DEVICE, >= casc_apply_seqsharded_workspace(m, p, q, L_loc, batch, N, world, mode, halo) bytes
 *     (derived weights, two state buffers of (2^Ne + L_loc) * batch * m elements with the halo
 *     rows in front, and the u halo row).
 *   Stream-ordered on compute_stream / comm_stream (distinct streams of the current device); no
 *   host synchronisation except inside the local transport's rendezvous (host threads wait for
 *   their neighbours to enqueue, never for the device).
 * Errors: CASC_ERR_ARG, CASC_ERR_DIM, CASC_ERR_WORKSPACE, CASC_ERR_UNSUPPORTED (m, p, q not
 *   multiples of 64, or world > 1 with a halo longer than L_loc: it would span several ranks),
 *   CASC_ERR_CUDA, CASC_ERR_NCCL (libnccl missing, or an NCCL call failed).
 * -------------------------------------------------------------------------------------- */
int casc_nccl_unique_id(void* id_out);
int casc_comm_init(void** comm, int rank, int world, const void* nccl_unique_id);
int casc_comm_init_local(void** comms, int world);
int casc_comm_destroy(void* comm);
int casc_comm_rank(const void* comm, int* rank, int* world);
/* halo: how the shard boundary is crossed (all three give the same y bit for bit)
 *   CASC_HALO_PER_STAGE  (BASELINE configs[3]) one exchange per step as above; compute = the shard.
 *   CASC_HALO_PEER       (fused) the step producing v^(k) stores the last 2^k rows
 *                        of its output ALSO into rank r+1's halo rows, from the GEMM epilogue over a
 *                        peer mapping (NVLink), tile by tile as they are produced; the transport
 *                        only orders the ranks with 1-byte tokens (ready: rank r-1's producing step
 *                        finished; consumed: rank r+1 has read the halo rows about to be
 *                        overwritten). NCCL ranks map rank r+1's ws through CUDA IPC once per call
 *                        (ws must be cudaMalloc memory; else every rank returns
 *                        CASC_ERR_UNSUPPORTED); emulated ranks store into each other's ws directly.
 *                        Needs the CTA-pair GEMMs (m a multiple of 256 in bf16, of 128 in fp32) and
 *                        halo rows produced by the interior launch (2^k * batch <= L_loc * batch -
 *                        boundary rows), else CASC_ERR_UNSUPPORTED.
 *   CASC_HALO_ONESHOT_U one exchange of Hu = 2^(Ne+1) - 1 time rows of u from rank
 *                        r-1 (the cascade is a polynomial of degree 2^(Ne+1) - 1 in the shift,
 *                        PAPER.md:137-141), then the cascade runs on the window [l0 - Hu, l0 + L_loc)
 *                        with no further communication: Hu / L_loc extra rows of work (E4 at 8 ranks:
 *                        3.1%). Requires Hu <= L_loc when world > 1.
 * (each output row is computed by the same operations in every mode). */
enum { CASC_HALO_PER_STAGE = 0, CASC_HALO_ONESHOT_U = 1, CASC_HALO_PEER = 2 };
size_t casc_apply_seqsharded_workspace(int m, int p, int q, int64_t L_loc, int batch, int N, int world, int mode,
                                       int halo);
int casc_apply_seqsharded(void* comm, int m, int p, int q, int64_t L_loc, int batch, int N, int N_max, int mode,
                          int halo, const void* pack, const double* Bbar, const double* C, const double* D,
                          const void* u_loc, void* y_loc, void* ws, size_t ws_bytes, void* compute_stream,
                          void* comm_stream);

/* Number of kernel launches the last successful apply/powers call on this host thread
 * enqueued (bench evidence for "gpu_launches"). */
int casc_last_launch_count(void);

/* ----------------------------------------------------------------------------------------
 * Optional per-kernel-class timing (measurement support, bench.py). When enabled on the
 * calling host thread, every launch the library enqueues is bracketed by CUDA events
 * recorded on its own stream and tagged with its kernel class and ALGORITHMIC bytes / flops.
 * casc_profile_read synchronises the recorded events of one class and returns the launch
 * count, summed device milliseconds, bytes and flops (any pointer may be NULL).
 * casc_profile_reset drops all records. Classes: 0 .. casc_profile_num_classes()-1, named by
 * casc_profile_class_name (static strings).
 * -------------------------------------------------------------------------------------- */
int casc_profile_enable(int on);
int casc_profile_reset(void);
int casc_profile_num_classes(void);
const char* casc_profile_class_name(int cls);
int casc_profile_read(int cls, int* launches, double* ms, double* bytes, double* flops);
/* The EXECUTED work of the same records (summed): the HBM bytes the schedule run moves and the
 * math-pipe flops it issues (3xTF32 counts three tf32 products; skipped zero blocks are not
 * counted); pipe: 0 none, 1 tf32, 2 bf16 (kind::f16: bf16 or fp16 operands, the same rate),
 * 3 fp64, 4 fp32 (CUDA cores) -- the peak to judge them by. */
int casc_profile_read_exec(int cls, double* exec_bytes, double* exec_flops, int* pipe);

/* ----------------------------------------------------------------------------------------
 * Hardware self-test of the tensor-core building block (diagnostics; used by tests/):
 *   D[128][64] = A[off:off+128][0:64] . B[0:64][0:64]^T on tcgen05 kind::tf32, fp32 accumulate,
 *   operands staged in shared memory in the K-major no-swizzle layout the cascade kernels use.
 *   prep: 0 raw fp32 bits, 1 pre-truncated to tf32, 2 rounded (rna) to tf32.
 *   A DEVICE float [144][64], B DEVICE float [64][64], D DEVICE float [128][64]; 0 <= off <= 16.
 * -------------------------------------------------------------------------------------- */
int casc_selftest_umma(int prep, int off, const float* A, const float* B, float* D, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CASCADE_B200_H */
