/*
 * nslct.h -- C ABI of the B200-native 2D nonseparable discrete linear canonical
 * transform (2D NsDLCT) of arxiv 1707.03688 ("PAPER.md").
 *
 * The problem (Eq. Intro08): given N x N complex
 * samples g[m,n] = g(m dx, n dx) and a valid ABCD matrix (Eq. Intro04, PAPER.md:27-58;
 * validity Eq. Intro12), compute N x N samples G[p,q] ~ G(p dx, q dx)
 * of its 2D NsLCT.  For det B != 0 the library evaluates the paper's fast HA-NsDLCT
 *     O = CM((D'-I)B'^-1) CC(B') CM(B'^-1(A-I)) CC(H)          (Eq. HA28)
 * or its CC-CM-CC-CM mirror (Eq. CCCMCCCM40), chosen by the
 * reversible dispatch of Eq. Reversible08 (reading R7),
 * where CC(B) = F^-1 CM(-B) F (Eq. BasicCC20) and F is the 2D DFT of
 * Eq. BasicDFT16 with F^-1 its exact inverse (reading R3).  For B = 0 it
 * evaluates Eq. Intro20 as chirp x bilinear affine resampling
 * (Eq. BasicAffine12/16).
 *
 * Conventions (readings R1/R2):
 *   - centered indices m, n, p, q in [-N/2, N/2-1], stored at array index m + N/2;
 *   - data layout [batch][N][N], row index = m (x), column index = n (y, contiguous);
 *   - input and output on the same grid dx (Delta_u = Delta_x);
 *     the frequency grid of the CC middle chirp has spacing 2 pi / (N dx);
 *   - complex numbers interleaved (re, im): NSLCT_C64 = 2 x float, NSLCT_C128 = 2 x double;
 *   - the output carries no extra normalisation: the transform is unitary.
 *
 * Errors: every call returns an nslct_status and never aborts; a thread-local message
 * is available from nslct_last_error().  The inverse transform is nslct_plan() on
 * M^-1 = (D^T, -B^T; -C^T, A^T) (Eq. CCCMCCCM20); with the reversible dispatch,
 * exec(plan(M^-1)) o exec(plan(M)) is the identity to rounding.
 */
#ifndef NSLCT_H
#define NSLCT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSLCT_ABI_VERSION 4

typedef enum { NSLCT_C64 = 0, NSLCT_C128 = 1 } nslct_dtype;

typedef enum {
  NSLCT_OK = 0,
  NSLCT_E_ARG = 1,             /* null/misaligned pointer, bad batch/dtype/option            */
  NSLCT_E_NOT_SYMPLECTIC = 2,  /* an Eq. Intro12 residual exceeds 1e-10                       */
  NSLCT_E_NO_DECOMP = 3,       /* no feasible H with |det B'| > 1e-8 max(1,|B'|^2) (reading R5) */
  NSLCT_E_UNSUPPORTED_N = 4,   /* N outside [2, 4096] and not a power of two <= 16384 (c128:
                                  8192); or no on-chip kernel for NSLCT_SCHEDULE_ON_CHIP     */
  NSLCT_E_CUDA = 5,            /* a CUDA launch/copy/allocation call failed (see last_error)  */
  NSLCT_E_NCCL = 6,            /* NCCL unavailable, or an NCCL call of the slab mode failed     */
  NSLCT_E_OOM = 7              /* device allocation of the plan's scratch failed              */
} nslct_status;

typedef struct nslct_plan_s* nslct_plan_t;

/* plan variants */
enum { NSLCT_VARIANT_HA = 0,       /* H by the HA objective of Eq. HA24, search of reading R5     */
       NSLCT_VARIANT_LC = 1,       /* H = (h,0;0,0) or (0,0;0,h) of Eq. LC08/LC10, HA fallback     */
       NSLCT_VARIANT_FIXED_H = 2,  /* H given in nslct_opts.h_fixed (form I: H of M; form II:
                                      H~ = the form-I H of M^-1), e.g. to reproduce another plan */
       NSLCT_VARIANT_DING = 3      /* Ding's method, the paper's comparison system (Eq. Ding12,
                                      PAPER.md:556-568): CM(B^-1 A), the 2D DFT
                                      of the input zero-padded to 2N x 2N ("two-times
                                      upsampling"), bilinear affine B^-T from that frequency grid
                                      to the output grid, CM(D B^-1); kind 3, 3 launches.  Needs
                                      det B != 0 (B = 0 takes the Eq. Intro20 path as for every
                                      variant); 2N a power of two <= 16384 (c128: 8192) or
                                      2N <= 4096; no slab or padded form.  Not unitary: an
                                      approximation of the continuous NsLCT, like the paper's. */
};
/* dispatch policies */
enum { NSLCT_DISPATCH_REVERSIBLE = 0,  /* Eq. Reversible08 + odd tie key (reading R7) */
       NSLCT_DISPATCH_FORM_I = 1        /* always CM-CC-CM-CC (reading R8)            */
};

typedef struct {
  double dx;          /* sample spacing dx = dy = du = dv; <= 0 selects sqrt(2 pi / N)  */
  int variant;        /* NSLCT_VARIANT_*                                                */
  int dispatch;       /* NSLCT_DISPATCH_*                                               */
  double h_fixed[3];  /* (h11, h22, h12) for NSLCT_VARIANT_FIXED_H                      */
  int device;         /* CUDA device ordinal for the plan's buffers; -1 = current       */
  int profile;        /* 1: record per-pass CUDA events in nslct_exec (nslct_pass_ms)   */
  int schedule;       /* NSLCT_SCHEDULE_*: how a batched plan's passes are launched      */
  int n_in;           /* fused zero-padding:
                         0 = none; else 1 <= n_in <= n is the side of the INPUT images,
                         [batch][n_in][n_in], placed on the n x n grid with every sample
                         keeping its centred coordinate (rows/columns [n/2 - n_in/2,
                         n/2 - n_in/2 + n_in)), zeros elsewhere; same dx; the output is
                         [batch][n][n].  Padded plans cannot run in place and have no
                         row-slab form.                                                    */
  int kernels;        /* NSLCT_KERNELS_*: which kernel family runs the line passes        */
  int host_chunk_kb;  /* nslct_exec_host pipeline chunk (KiB); 0 = min(64 MiB, batch bytes / 8) */
  void* comm;         /* NULL: single GPU.  An nslct_comm_t from nslct_comm_init: the plan is
                         ONE n x n transform row-slab sharded over the communicator's ranks
                         (SURVEY.md §8(e)); `batch` must be 1, and nslct_exec runs every pass
                         and every all-to-all on its stream (see nslct_exec).               */
  int exchange_chunks;/* slab mode: chunks per pass whose all-to-all overlaps the next
                         chunk's compute (1, 2, 4 or 8; 0 = 2)                            */
  int exchange;       /* slab mode: NSLCT_EXCHANGE_*                                        */
  int reserved[4];
} nslct_opts;
/* how a comm plan moves data between passes */
enum { NSLCT_EXCHANGE_NCCL = 0,   /* NCCL grouped send/recv of each chunk's sub-blocks, on a
                                     plan-owned stream, overlapping the next chunk's compute */
       NSLCT_EXCHANGE_PEER = 1    /* the transposing pass stores row-block s of its output
                                     straight into rank s's receive buffer over NVLink (CUDA
                                     IPC peer mappings made at plan time; nranks <= 8), one
                                     stream-ordered cross-rank barrier (a 4-byte NCCL
                                     all-reduce) after each such pass: no separate exchange
                                     phase and no send buffer                                */
};
/* kernel families (all compute the same operator) */
enum { NSLCT_KERNELS_AUTO = 0,     /* the specialised kernels where they exist: persistent
                                      TMA pipe (c64, N = 1024..4096), TMA-pipelined cluster
                                      pairs (c64, N = 8192), cluster pairs (c64, N = 16384),
                                      on-chip (see schedule)                                 */
       NSLCT_KERNELS_GENERIC = 1   /* one CTA per group of lines everywhere (A/B reference)  */
};
/* schedules of a batched plan (all compute the same operator) */
enum { NSLCT_SCHEDULE_AUTO = 0,        /* the on-chip kernel for N <= 64 (measured faster at
                                          every batch size: tools/schedule_sweep.py,
                                          DESIGN.md §6.8), else one launch per pass         */
       NSLCT_SCHEDULE_LINE_PASSES = 1, /* always one launch per pass                        */
       NSLCT_SCHEDULE_ON_CHIP = 2      /* the on-chip kernel wherever one exists: c64 N <= 256
                                          (N = 256: 4-CTA cluster), c128 N <= 128 (N = 128:
                                          4-CTA cluster); NSLCT_E_UNSUPPORTED_N otherwise     */
};

/* Fill *opts with the defaults (dx = sqrt(2 pi/N), HA, reversible, current device). */
void nslct_opts_default(nslct_opts* opts);

/* Build a plan for `batch` transforms of size n x n with ABCD matrix abcd (row-major
 * 4x4: [[a11 a12 b11 b12],[a21 a22 b21 b22],[c11 c12 d11 d12],[c21 c22 d21 d22]],
 * PAPER.md:46-51).  Host-side planning (validation, dispatch, H search) plus device
 * allocation of twiddle tables and one scratch buffer of batch*n*n complex elements on
 * the selected device.  The plan owns everything it allocates; free with nslct_destroy.
 * n: a power of two in [32, 16384] (c128: <= 8192) runs the radix-16 line FFTs; any
 * other n in [2, 4096] (odd n included: the paper's N = 165 + dN) runs
 * every line DFT by Bluestein's identity with power-of-two FFTs of length
 * 2^ceil(log2(2n-1)), same operator, same layouts (nslct_plan_desc.fft_len). */
nslct_status nslct_plan(nslct_plan_t* plan, int64_t n, const double abcd[16], int64_t batch,
                        nslct_dtype dtype);
nslct_status nslct_plan_ex(nslct_plan_t* plan, int64_t n, const double abcd[16], int64_t batch,
                           nslct_dtype dtype, const nslct_opts* opts);

/* Enqueue the transform of `batch` images on `cuda_stream` (a cudaStream_t; NULL = the
 * legacy default stream).  in/out: DEVICE pointers to [batch][n][n] interleaved complex
 * (in: [batch][n_in][n_in] for a zero-padding plan), 16-byte aligned, owned by the
 * caller; in == out is allowed (not for a padding plan).  Asynchronous and
 * stream-ordered: no host synchronisation, no allocation.  At most one exec per plan in
 * flight (the plan's scratch is shared).  Errors: E_ARG (null/misaligned), E_CUDA.
 *
 * Slab plans (opts.comm set): in/out are this rank's row slab [L][n], L = n/nranks (rows
 * [rank*L, (rank+1)*L) of the input and of the output).  Every rank calls nslct_exec with
 * its slab; the call enqueues the n_passes passes and, between consecutive passes, the
 * all-to-all that re-shards row slabs into column slabs and back (the distributed form of
 * the transposes the single-GPU passes fold into their stores): NCCL
 * grouped send/recv of L x L/c sub-blocks, chunk by chunk (c = opts.exchange_chunks), on
 * a plan-owned stream ordered after each chunk's pass, so chunk k's exchange overlaps
 * chunk k+1's compute -- or, with opts.exchange = NSLCT_EXCHANGE_PEER, fused into the
 * passes' stores to the peers' receive buffers.  Creating a comm plan is collective (every
 * rank of the communicator, same arguments: the PEER mode exchanges IPC handles).
 * Errors: additionally E_NCCL. */
nslct_status nslct_exec(nslct_plan_t plan, const void* in, void* out, void* cuda_stream);

/* Same transform from HOST memory: copies host_in -> device, runs the passes, copies the
 * result back to host_out, and returns only when host_out holds the result.  The batch
 * runs as a pipeline of chunks of whole images (at most 64 MiB and about 1/8 of the batch
 * each; opts.host_chunk_kb overrides): the host->device copy of chunk i+1 (on a plan-owned
 * copy stream), the
 * passes of chunk i (on cuda_stream) and the device->host copy of chunk i-1 (a second
 * plan-owned copy stream) overlap, so a large batch costs about one PCIe direction, not
 * both plus the compute.  The copies start after the work already queued on cuda_stream.
 * host buffers [batch][n][n] complex (host_in [batch][n_in][n_in] for a padding plan;
 * pinned memory gives full copy speed and overlap).
 * Device staging buffers, copy streams and events are created on the first call and
 * owned by the plan.  Errors: E_ARG (null pointers, slab plan, or -- for a zero-padding
 * plan, whose output chunks are larger than its input chunks -- overlapping host_in /
 * host_out ranges), E_CUDA, E_OOM. */
nslct_status nslct_exec_host(nslct_plan_t plan, const void* host_in, void* host_out,
                             void* cuda_stream);

/* Row-slab mode: ONE n x n transform sharded over nranks processes (one
 * per GPU) as row slabs of L = n/nranks rows; rank `rank` holds rows [rank*L, (rank+1)*L)
 * of the input and of the output, row-major [L][n].  The transform runs as n_passes
 * passes (nslct_plan_info); between consecutive passes the CALLER performs one all-to-all
 * of nranks equal blocks of L*L complex elements (e.g. NCCL through torch.distributed
 * all_to_all_single): the send buffer is the previous pass's `out`, laid out [n][L] =
 * nranks row-blocks of [L][L] (block s goes to rank s), and the receive buffer (block
 * from rank s at element offset s*L*L) is the next pass's `in`.  This exchange is the
 * distributed form of the transposes the single-GPU passes fold into their stores.  The
 * element order INSIDE a block is the library's (sub-blocks of opts.exchange_chunks
 * producer-line chunks; inside them plain transposed, or, for complex64, 16-byte
 * interleaved line pairs at n = 8192 and 8-byte interleaved line pairs at n = 16384:
 * DESIGN.md §7); the exchange must move whole blocks unchanged.
 * Requires B != 0 (the B = 0 gather has no slab form), nranks | n, and L a multiple of
 * the kernel's lines per CTA (L >= 16 suffices for n >= 4096).  The plan allocates no
 * scratch: the caller owns all buffers (each n*L complex elements).  Errors: as
 * nslct_plan_ex, E_ARG for bad nranks/rank/L. */
nslct_status nslct_plan_slab(nslct_plan_t* plan, int64_t n, const double abcd[16], int nranks,
                             int rank, nslct_dtype dtype, const nslct_opts* opts);

/* Run ONE pass (0 <= pass < n_passes) of a plan on `cuda_stream`: for a slab plan, the
 * pass of this rank's slab (layouts above); for a batched plan, pass k of nslct_exec
 * with the batched layouts (in/out are then the plan-documented intermediates; mainly
 * for debugging).  Asynchronous, no allocation.  Errors: E_ARG, E_CUDA. */
nslct_status nslct_exec_pass(nslct_plan_t plan, int pass, const void* in, void* out,
                             void* cuda_stream);

/* Row-slab pass with the all-to-all FUSED into its store (SURVEY.md §8(e) stretch): pass
 * `pass` (a transposing pass, 0 <= pass < n_passes - 1) of this rank's slab writes
 * row-block s of its [n][L] output straight into peer_out[s] -- a device buffer of rank s
 * (CUDA peer / NVLink memory, e.g. a torch symmetric-memory buffer), n*L elements -- at
 * element offset rank*L*L: exactly what the all_to_all_single of nslct_exec_pass would have
 * left in rank s's receive buffer, so the next pass reads it unchanged.  n_peers must equal
 * nranks (<= 8).  The CALLER orders the exchange: every rank's pass k must have finished
 * reading the buffers it is about to overwrite (double-buffer the receive buffers across
 * passes) and a cross-rank barrier must separate pass k's stores from pass k+1's reads.
 * Asynchronous on cuda_stream; no allocation.  Errors: E_ARG, E_CUDA. */
nslct_status nslct_exec_pass_peer(nslct_plan_t plan, int pass, const void* in, void* const* peer_out,
                                  int n_peers, void* cuda_stream);

/* ---- multi-GPU communicator (slab mode) ----------------------------
 * NCCL is loaded at run time (dlopen of libnccl.so.2: the copy already mapped into the
 * process, e.g. PyTorch's, else the system one); the library does not link it.  One
 * process per GPU: rank 0 calls nslct_comm_unique_id and distributes the 128 bytes (e.g.
 * through torch.distributed), then every rank calls nslct_comm_init with the CUDA device
 * it will run on current.  Errors: E_NCCL (library not found, NCCL error), E_ARG. */
typedef struct nslct_comm_s* nslct_comm_t;
nslct_status nslct_comm_unique_id(uint8_t unique_id[128]);
nslct_status nslct_comm_init(nslct_comm_t* comm, const uint8_t unique_id[128], int rank, int nranks);
/* rank / number of ranks of a communicator */
nslct_status nslct_comm_info(nslct_comm_t comm, int* rank, int* nranks);
/* Free the communicator (after every plan using it has been destroyed).  NULL is a no-op. */
nslct_status nslct_comm_destroy(nslct_comm_t comm);

/* The inverse transform's matrix M^-1 = (D^T, -B^T; -C^T, A^T) of Eq. CCCMCCCM20
 * (it inverts any matrix satisfying Eq. Intro12), row-major 4x4 as in
 * nslct_plan.  out may alias abcd.  Errors: E_ARG (null pointer). */
nslct_status nslct_inverse_matrix(const double abcd[16], double out[16]);

typedef struct {
  int kind;                    /* 0 = B=0 (Eq. Intro20), 1 = form I (Eq. HA28), 2 = form II,
                                  3 = Ding (Eq. Ding12; Q[0] = B^-1 A, Q[4] = D B^-1)          */
  int variant;                 /* variant actually used (LC falls back to HA: PAPER.md:840)  */
  int lc_axis;                 /* 0 none, 1 = H=(h,0;0,0) (x), 2 = H=(0,0;0,h) (y)            */
  int n_passes;                /* device passes per transform: 5 (HA, LC with x-axis H),      */
                               /* 3 (LC with y-axis H; Ding: two line passes
                                  of length 2N + the affine gather), 1 (B=0)                  */
  double H[3], Bp[3], P2[3], P4[3];  /* form-I plan of M (form I) or of M^-1 (form II):
                                        (q11, q22, q12) of H, B', P2=B'^-1(A-I), P4=(D'-I)B'^-1 */
  double Q[5][3];              /* the executed chirps, application order:
                                  CM_space(Q0) F CM_freq(Q1) F^-1 CM_space(Q2) F CM_freq(Q3)
                                  F^-1 CM_space(Q4); (q11, q22, q12)                        */
  double dx;                   /* sample spacing used                                         */
  double objective;            /* J(H) of Eq. HA24                                            */
  double sym_residual;         /* max Eq. Intro12 residual of the input matrix                */
  double recomposition_residual; /* |product of stage matrices - M|_max                        */
  double dispatch_key;         /* s(M) of reading R7                                          */
  int n_launches;              /* kernel launches per nslct_exec: 1 with on_chip, else
                                  n_passes (0 from nslct_plan_describe: no device chosen)     */
  int on_chip;                 /* 1: the whole transform runs in one kernel per image, the
                                  image held in shared memory (see
                                  NSLCT_SCHEDULE_*); nslct_exec_pass still runs line passes  */
  int fft_len;                 /* FFT length per line: N for a power-of-two N; for any other
                                  N the line DFTs run by Bluestein's chirp-z identity with
                                  FFTs of length 2^ceil(log2(2N-1)) (>= 32); 0 for B = 0   */
  int n_in;                    /* input side (== n unless the plan zero-pads)                 */
} nslct_plan_desc;

nslct_status nslct_plan_info(nslct_plan_t plan, nslct_plan_desc* out);

/* Host-only dry run of nslct_plan_ex: validation, dispatch and H search only, no CUDA call
 * and no allocation; fills *out as nslct_plan_info would.  n only selects the default dx.
 * Same error codes as nslct_plan_ex (except E_CUDA / E_OOM, which cannot occur). */
nslct_status nslct_plan_describe(int64_t n, const double abcd[16], const nslct_opts* opts,
                                 nslct_plan_desc* out);

/* Per-pass device times (ms), averaged over every nslct_exec of a plan built with
 * opts.profile = 1 since the previous call (events recorded on the exec stream between
 * passes).  Synchronises on those events, then resets the average.  ms must hold
 * n_launches floats; *n_written receives n_launches (one value for an on-chip plan). */
nslct_status nslct_pass_ms(nslct_plan_t plan, float* ms, int capacity, int* n_written);

/* Measured FP32 FMA throughput of `device` (TFLOP/s, 2 flops per FFMA): a calibration
 * kernel of independent FFMA chains on every SM, best of 3 timed launches (~ms each).  The
 * ALU ceiling reported next to the HBM roofline.  Synchronous.
 * Errors: E_ARG, E_CUDA. */
nslct_status nslct_fp32_peak(int device, double* tflops);

/* Free the plan and everything it owns (device-synchronises its buffers). NULL is a no-op. */
nslct_status nslct_destroy(nslct_plan_t plan);

/* Thread-local text of the last error on this thread ("" if none). */
const char* nslct_last_error(void);

/* NSLCT_ABI_VERSION of the loaded library. */
int nslct_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NSLCT_H */
