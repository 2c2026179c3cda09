/*
 * tn.h — C ABI of the B200-native stem-path contraction library (libtn.so).
 *
 * The operation (PAPER.md = arXiv 2407.00769, P:n = line n):
 *   Contract one sliced subtask of a random-quantum-circuit tensor network along a contraction
 *   tree whose stem path dominates the cost ("Stem Type / Split Type / Common Type";
 *   P:228).  Slicing fixes sliced edges to the bits of a slice id.  Each stem
 *   step is a pairwise contraction C = sum_delta A*B (Eq. 3) with the remaining indices
 *   of Eq. 4, executed as a mode permutation of the stem tensor plus a complex GEMM;
 *   in complex-half it runs as ONE real fp16 GEMM on tcgen05 via the Eq. 6 embedding
 *   (A read as interleaved (re,im), B padded to [[Re,-Im],[Im,Re]]), fp32 accumulation.
 *   The two stem buffers are the paper's static double buffers.
 *
 * Conventions
 *   - Every entry point returns int status (TN_OK = 0 or a negative TN_E_* code) and never lets a
 *     C++ exception cross the ABI.  tn_last_error() returns a thread-local message for the last
 *     failing call on this thread.
 *   - Pointers named d_* are DEVICE pointers; h_* are HOST pointers.  Device buffers are always
 *     caller-owned and only lent for the duration of a call (asynchronous calls: until the stream
 *     work completes).  The library owns tn_plan / tn_comm objects and frees them in *_free.
 *   - `stream` is a cudaStream_t passed as void*.  Asynchronous calls enqueue work on it and do
 *     not synchronise unless stated.
 *   - No CPU fallback exists: without a CUDA device the compute calls return TN_E_CUDA.
 */
#ifndef TN_H_
#define TN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TN_API __attribute__((visibility("default")))
#else
#define TN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TN_OK = 0,
  TN_E_INVALID = -1,     /* bad argument, inconsistent plan (dims, labels, tree), slice id range */
  TN_E_PARSE = -2,       /* malformed plan JSON */
  TN_E_INFEASIBLE = -3,  /* plan cannot run in the given configuration (capacity, shard modes) */
  TN_E_CAPACITY = -4,    /* caller buffers too small */
  TN_E_CUDA = -5,        /* CUDA runtime/driver error (incl. no device) */
  TN_E_NCCL = -6,        /* NCCL error */
  TN_E_UNSUPPORTED = -7  /* valid request this build does not implement */
};

/* stem compute dtype */
enum { TN_CHALF = 0,   /* complex-half: interleaved fp16 (re,im), fp32 accumulation */
       TN_CFLOAT = 1   /* complex64: interleaved fp32, fp32 SIMT FMA (reference-precision path) */ };

/* mode-swap payload codec (Eq. 1, Table 1):
 *   TN_COMM_INT8 / TN_COMM_INT4: per-block groups of cfg.comm_group reals (power of two >= 16), exp 1
 *   TN_COMM_INT8_TENSOR: the paper's Table 1 int8 preset: one group per destination chunk
 *     (the "entire tensor" a peer receives; groups never straddle destinations), exp 0.2 (C-A10) */
enum { TN_COMM_FP16 = 0, TN_COMM_INT8 = 1, TN_COMM_INT4 = 2, TN_COMM_INT8_TENSOR = 3 };

typedef struct tn_plan tn_plan;
typedef struct tn_comm tn_comm;

typedef struct {
  int32_t dtype;             /* TN_CHALF | TN_CFLOAT */
  int32_t stem_min_log2;     /* stem steps begin at the first stem node holding >= 2^this
                                elements; everything before is common type.  <0: 20.
                                If that node holds > 2^(this+2), the entry moves back along the
                                stem (to internal nodes >= 2^(this-8)) until it does not. */
  int32_t comm_codec;        /* TN_COMM_* for sharded mode swaps (ignored at world size 1) */
  int32_t comm_group;        /* quantisation group in reals (int8/int4), e.g. 128 */
  uint64_t stem_capacity_bytes; /* bytes of EACH stem buffer the caller will lend; 0 = no check */
  int32_t split_log2;        /* split-type tail: 2^split_log2 chunks, each fixing
                                split_log2 open legs that stay the outermost local modes of the
                                tail (never shard modes; a sharded stem chunks every rank's shard,
                                and a mode swap inside the tail is TN_E_INFEASIBLE).  0 = no split.
                                -1 = auto, "determined by the current remaining capacity"
                                (reading C-A19): the smallest power of two whose lowering fits
                                stem_capacity_bytes (capacity 0: no split); tn_plan_load returns
                                TN_E_CAPACITY when no chunk count fits.  tn_plan_info.split_chunks
                                reports the count chosen. */
  int32_t layout_policy;     /* 0 (default): output = kept ++ new (TMA-store epilogue) plus a
                                permutation pass when the next step's modes are not innermost;
                                2: each GEMM writes its output with the next step's contracted
                                modes innermost (scatter epilogue, no permutation passes);
                                1: scatter when its stores are >= 64 B contiguous, else as 0;
                                3: as 0, but a GEMM writes C[n][m] (new modes outermost, a
                                transposed store whose warps write 128 contiguous bytes) when that
                                puts more of the next step's contracted modes innermost */
  int32_t quant_from_pct;    /* int8/int4 swaps only at stem steps >= this percentage of the path
                                ("quantify in the later stages"); earlier swaps send
                                fp16.  Negative: 65 (the sub-sliced C3 at 8 ranks keeps the
                                north_star 5e-2 bound with int8 swaps from 65 %, not from 50 %) */
  int32_t virtual_world;     /* > 1 with comm == NULL: lower the plan for that many ranks
                                (host-only inspection of the shard/swap schedule) */
  int32_t no_gather;         /* 0 (default): a permutation before a tensor-core step whose two
                                innermost modes are contracted is fused into the GEMM's A load
                                (gathered cp.async, no permutation pass); 1: always a pass */
  int32_t no_fuse_swap_quant; /* 0 (default): a quantised mode swap whose sender permutation keeps
                                the innermost log2(comm_group/2) modes in place quantises straight
                                from the unpermuted stem (tn_permute_quant_f16, no permutation
                                pass); 1: permutation pass, then the codec */
  int32_t recompute;         /* 1: recomputation on halves: the stem
                                is halved along one open leg (a free mode of the largest stem
                                tensor) right before the step that produces that tensor; the rest
                                of the path runs twice, once per half, inside the two stem buffers,
                                and the halves are concatenated (split machinery with 2 chunks, so
                                tn_split_contract runs the halves).  Peak stem bytes halve when the
                                largest tensor lies in the recomputed region.  Needs split_log2 = 0;
                                no mode swap may fall into the recomputed region ("there is no data
                                communication").  0: off */
  int32_t no_fused_swap;     /* 0 (default): an fp16 mode swap right after a tcgen05 GEMM step is
                                done by that GEMM's epilogue — each output tile is TMA-stored
                                straight into the buffer of the rank that owns it after the swap
                                (NVLink peer memory: CUDA IPC between processes, plain pointers
                                between loopback ranks), when the swapped modes are tile-constant
                                (m bits >= 7, n bits >= 5); bit-identical to the exchange.
                                1: every swap through the transport (NCCL send/recv) */
} tn_config;

/* Caller-owned device buffers lent to a call (P:18-22 double buffering). */
typedef struct {
  void* d_stem[2];           /* the two static stem buffers */
  uint64_t stem_bytes;       /* size of EACH stem buffer */
  void* d_ws;                /* workspace: leaves, common-type tensors, padded B_P, scale slots */
  uint64_t ws_bytes;
} tn_buffers;

typedef struct {
  uint64_t ws_bytes;         /* workspace bytes tn_stem_contract needs */
  uint64_t stem_bytes;       /* bytes each stem buffer needs (max stem tensor, this dtype) */
  uint64_t n_slices_log2;    /* |sliced| : the network has 2^this independent subtasks */
  uint64_t n_stem_steps;     /* stem steps executed on the stem buffers */
  uint64_t n_permutes;       /* stem steps that need a standalone permutation pass */
  uint64_t n_common;         /* common-type (branch) contractions per slice */
  double stem_flops;         /* 8 * sum b*M*K*N over stem steps (reading C-A21) */
  double total_flops;        /* 8 * complex MACs of the whole slice (common + stem) */
  double stem_bytes_alg;     /* algorithmic HBM bytes of the stem GEMMs (A read + C write) */
  double perm_bytes;         /* bytes moved by standalone permutation passes */
  uint64_t n_open;           /* open legs: the result has 2^n_open amplitudes */
  uint64_t max_stem_log2;    /* log2 elements of the largest stem tensor */
  uint64_t h2d_bytes;        /* bytes tn_plan_upload copies host->device */
  uint64_t split_chunks;     /* chunk count of the split-type tail (1 = none) */
  uint64_t n_launches;       /* kernels the last tn_stem_contract launched (0 before the first) */
  uint64_t n_sparse_legs;    /* sparse-state legs (plan "sparse_legs"): a subspace block holds
                                2^(n_open - n_sparse_legs) members */
} tn_plan_info;

TN_API const char* tn_last_error(void);
TN_API int tn_version(void);
/* Select the CUDA device for this thread's subsequent calls (libtn links its own CUDA runtime, so
 * the caller's framework-level device selection is not implied). */
TN_API int tn_set_device(int device);

/* Parse + validate + lower a plan (host only; no device work, no allocation on the device).
 * json: the plan JSON (tensors with labels/dims-2 complex128 data, open legs, SSA tree, sliced
 * labels, optional stem; see workload/make_plans.py).  cfg may be NULL (defaults).  comm: NULL for
 * one GPU.  Errors: TN_E_PARSE (syntax), TN_E_INVALID (label/dim/tree inconsistency, hyper-edge,
 * sliced open leg), TN_E_INFEASIBLE (largest stem exceeds cfg->stem_capacity_bytes). */
TN_API int tn_plan_load(const char* json, size_t len, const tn_config* cfg, tn_comm* comm, tn_plan** out);
TN_API int tn_plan_info_get(const tn_plan* p, tn_plan_info* info);
TN_API void tn_plan_free(tn_plan* p);

/* Copy the plan's leaf tensors (complex128 from the JSON, held in pinned host memory) into the
 * workspace as complex64, asynchronously on `stream`.  Must precede the first tn_stem_contract
 * with a given workspace; the end-to-end harness calls it every step (its H2D traffic). */
TN_API int tn_plan_upload(tn_plan* p, const tn_buffers* b, void* stream);

/* Run slice `slice_id` (bit j fixes sliced[j], reading C-A20; sliced labels beyond the 64th are
 * fixed to 0, so a plan with more than 64 sliced labels exposes its first 2^64 subtasks here):
 * common-type branch contractions,
 * Eq. 6 padding of every stem operand, then the stem steps (permutation + GEMM per step) in the
 * two stem buffers.  Asynchronous; result stays on the device.  TN_E_INVALID if
 * slice_id >= 2^|sliced|; TN_E_CAPACITY if the buffers are smaller than tn_plan_info says.
 * Single-rank plans: the slice id is written to the workspace by one kernel and the rest of the
 * call is a replay of a CUDA graph captured (on a library-owned stream) at the first call with a
 * given buffer set / timing flag; the graph is re-captured when either changes.  Buffers must
 * therefore stay allocated while the plan may replay them (free the plan first). */
TN_API int tn_stem_contract(tn_plan* p, const tn_buffers* b, uint64_t slice_id, void* stream);

/* Split-type tail: the last stem steps run on 2^split_log2 contiguous
 * chunks of the stem placed inside the two stem buffers.  No-op when the plan has no split tail.
 * Asynchronous. */
TN_API int tn_split_contract(tn_plan* p, const tn_buffers* b, void* stream);

/* Read the result, SYNCHRONOUS (writes host memory).
 * Dense (prefixes == NULL, n_sub == 0): h_amps receives 2 * 2^n_open doubles (interleaved re, im)
 * of the partial amplitudes a_s over the open legs in plan order (slowest first), unscaled exactly
 * by the accumulated power-of-two exponents (reading C-A8); top_idx (if not NULL) receives the k
 * most probable indices (ties -> smaller index, C-A23).
 * Sparse-state batch (Fig. 5; needs cfg.split_log2 = j > 0): prefixes[i] < 2^j selects a
 * correlated subspace = one value of the j split legs (bit j-1-t of the prefix <-> the t-th split leg
 * in plan order, i.e. in the order the legs appear in `open`; "split_modes" in tn_report_json lists
 * the legs in chunk order, which depends on the layouts); only those chunks of the tail are contracted.  h_amps receives
 * n_sub blocks of 2^(n_open-j) amplitudes (members = the other open legs in plan order); top_idx
 * receives n_sub*k member indices (post-selection; one rank: k = 1 on the device).
 * Sharded plans: every rank calls it (collective: the result blocks are gathered in rank order into
 * the workspace) and every rank receives the whole result.  Ties in top_idx always go to the smaller
 * member index in member order, whatever the storage layout (C-A23); NaN probabilities rank lowest.
 * Errors: TN_E_INVALID (k < 0, prefix >= 2^j), TN_E_UNSUPPORTED (prefixes without a split tail). */
TN_API int tn_sample_amplitudes(tn_plan* p, const tn_buffers* b, const uint64_t* prefixes, size_t n_sub,
                         double* h_amps, int k, uint64_t* top_idx, void* stream);

/* JSON report: per stem step geometry, permutation flag, flops, algorithmic bytes, and (after a
 * run with timing enabled) "ms": [common phase, (permutation, GEMM) per step..., final perm],
 * measured with CUDA events on the call's stream (synchronises on the last event).
 * *needed = bytes required incl. NUL. */
TN_API int tn_report_json(const tn_plan* p, char* buf, size_t cap, size_t* needed);
/* Enable CUDA-event timing of the phases of tn_stem_contract (events only, no host sync). */
TN_API int tn_set_timing(tn_plan* p, int enable);
/* Enable (default) or disable the CUDA-graph replay of tn_stem_contract (disabled: every launch
 * is issued eagerly on the caller's stream; also forced by the environment variable TN_NO_GRAPH). */
TN_API int tn_set_graph(tn_plan* p, int enable);

/* ---- kernel-level entry points (used by the parity tests; same kernels as the stem loop) ---- */

/* Mode permutation of a rank-n tensor with all dims 2 ("dimension reordering").
 * d_src/d_dst: 2^n elements of elem_bytes (4 = complex-half, 8 = complex64) each, must not
 * overlap.  perm[j] = source axis of destination axis j (numpy transpose semantics; axis 0 is
 * the slowest).  n <= 40. */
TN_API int tn_permute(void* d_dst, const void* d_src, int elem_bytes, int n, const int* perm, void* stream);

/* Complex-half stem GEMM, Eq. 6 as one real fp16 tcgen05 GEMM:
 *   C[m, n] = 2^e * sum_k A[m, k] B[k, n]   (complex; A, C interleaved fp16 (re,im) row-major)
 * d_bp: padded real B_P, fp16 [2N][2K] row-major (K-major): row (n,c), column (k,a) holds
 * c=0: (Re b, -Im b)[a], c=1: (Im b, Re b)[a] (reading C-A6).  The scale 2^e is chosen on the
 * device from *d_in_max (max |real component| of A) and *d_b_bound (max column 1-norm of B_P)
 * so that |C| <= 2^14; e is written to *d_exp.  *d_out_max receives max |real component| of the
 * scaled fp32 results before their fp16 rounding, as float bits (atomicMax; caller zeroes it; it
 * stays meaningful when cancellation makes the stored fp16 values underflow).  A negative *d_in_max
 * makes the launch return at once (the library's scale re-run uses that as "not needed").  Any of
 * the four scale pointers may be NULL: then e = 0 and no max is recorded.  K, N powers of two, M any.  K >= 4 runs on tcgen05 (for N < 8,
 * d_bp must hold 16 rows with rows 2N..15 zero); K < 4 runs on the SIMT kernel. */
TN_API int tn_gemm_chalf(void* d_c, const void* d_a, const void* d_bp, uint64_t M, uint32_t K, uint32_t N,
                  const float* d_in_max, const float* d_b_bound, uint32_t* d_out_max, int* d_exp,
                  void* stream);

/* tn_gemm_chalf with a strided (gathered) A: A[m, k] is the complex-half element at
 * d_a + sum_j bit_j(m) m_stride[j] + sum_j bit_j(k) k_stride[j] (complex elements; j = 0 is the
 * lowest bit).  This is the stem permutation fused into the GEMM load ("dimension
 * reordering").  M = 2^mlog >= 128, K = 2^klog >= 8, N a power of two; C row-major [M][N].  Any
 * strides: with k_stride[0] = 1, k_stride[1] = 2 the load moves 16-byte pieces (N-d TMA boxes or
 * cp.async), otherwise 4-byte cp.async pieces (coalesced when the 5 smallest strides among m bits
 * 0..6 and k bits 0..4 are 1, 2, 4, 8, 16).  Scale pointers as tn_gemm_chalf.  TN_E_INVALID
 * otherwise. */
TN_API int tn_gemm_chalf_gather(void* d_c, const void* d_a, const void* d_bp, int mlog, int klog, uint32_t N,
                                const int64_t* m_stride, const int64_t* k_stride, const float* d_in_max,
                                const float* d_b_bound, uint32_t* d_out_max, int* d_exp, void* stream);

/* Gather-batched complex-half GEMM (sparse-state contraction, P:533-537 and Fig. 5 bottom:
 * "obtain multiple tensors at specified positions through the indices Index_A and Index_B to form
 * A_I and B_I before performing matrix multiplication"):
 *   C[b] = 2^e A[index_a[b]] B[index_b[b]],  b < n_out,
 * one tcgen05 launch for the whole batch (A_I / B_I are never materialised: the TMA loads read the
 * indexed entries in place).  A: n_a entries of [M][K] complex-half (interleaved fp16, row-major,
 * entry a at element a*M*K); B_P: n_b blocks of fp16 [2N][2K] (tn_gemm_chalf's B_P layout, block j at
 * element j*4*N*K); C: n_out entries of [M][N] complex-half.  index_a / index_b: DEVICE int32 arrays
 * of n_out entries (< n_a / < n_b; not checked on the device).  M a multiple of 128, K >= 4 and N >= 8
 * powers of two; the scale pointers as tn_gemm_chalf (one exponent for the whole batch). */
TN_API int tn_gemm_chalf_batched(void* d_c, const void* d_a, const void* d_bp, uint64_t M, uint32_t K, uint32_t N,
                                 uint64_t n_out, const int32_t* d_index_a, const int32_t* d_index_b, uint64_t n_a,
                                 uint64_t n_b, const float* d_in_max, const float* d_b_bound, uint32_t* d_out_max,
                                 int* d_exp, void* stream);
/* Padded 2-d index variant (Fig. 5 top: "we use the input tensor A directly ... padding
 * Index_B to a new 2d-index whose size is m_a*m_r ... excess positions are replaced with -1 ...
 * C_P = A x B_P"): C_P[a] = A[a] [B[t(a,0)] | B[t(a,1)] | ... | B[t(a,m_r-1)]] for a < n_a, with
 * t(a,r) = table[a*m_r + r] (DEVICE int32, row-major [n_a][m_r]); t < 0 gives a zero block (its MMA
 * is skipped).  C_P: n_a entries of [M][m_r*N] complex-half; the valid products are the blocks
 * with t >= 0 (C is C_P "flattened ... then extract valid tensors in it").  Shapes as above, and
 * N >= 32 when m_r > 1. */
TN_API int tn_gemm_chalf_padded(void* d_c, const void* d_a, const void* d_bp, uint64_t M, uint32_t K, uint32_t N,
                                uint64_t n_a, const int32_t* d_table, int m_r, uint64_t n_b, const float* d_in_max,
                                const float* d_b_bound, uint32_t* d_out_max, int* d_exp, void* stream);

/* Complex64 stem GEMM (fp32 SIMT): C[M,N] = A[M,K] B[K,N], all interleaved complex64 row-major. */
TN_API int tn_gemm_cfloat(void* d_c, const void* d_a, const void* d_b, uint64_t M, uint32_t K, uint32_t N,
                   void* stream);

/* The stem permutation of a step stored as [M >> ma][K][2^ma] (its 2^ma innermost modes are kept
 * modes, its contracted modes come next: P:534's "dimension reordering" when the contracted modes
 * sit in the middle of the stored order) folded into the operand layout instead of a pass:
 *   C[m, n] = 2^e sum_k A[m, k] B[k, n],  A[m, k] at element ((m >> ma) K + k) 2^ma + (m & (2^ma-1)),
 * computed as the real GEMM over rows (m, c) of an MN-major operand on the CTA-pair tcgen05 kernel
 * (same 4 M K N real MACs as Eq. 6; the complex combination in the epilogue).
 * d_bpm = B' fp16 [2N][K] from tn_pad_b_mn.  C row-major [M][N] complex-half.  ma >= 7, M a
 * multiple of 128 with 2^ma <= M < 2^31, K >= 64 and N >= 64 powers of two; scale pointers as
 * tn_gemm_chalf.  TN_E_INVALID otherwise (also when the CTA-pair kernel is disabled, TN_TC2=0). */
TN_API int tn_gemm_chalf_mn(void* d_c, const void* d_a, const void* d_bpm, uint64_t M, uint32_t K, uint32_t N,
                            int ma, const float* d_in_max, const float* d_b_bound, uint32_t* d_out_max, int* d_exp,
                            void* stream);
/* B' for tn_gemm_chalf_mn: rows (n, 0) = Re B[:, n], (n, 1) = Im B[:, n] (fp16, k contiguous), from
 * complex64 B [K][N]; scale, *d_exp and *d_b_bound exactly as tn_pad_b. */
TN_API int tn_pad_b_mn(void* d_bpm, const void* d_b, uint32_t K, uint32_t N, float* d_b_bound, int* d_exp,
                       void* d_scratch /* >= 16 bytes */, void* stream);

/* Build B_P (fp16 [2N][2K]) from complex64 B [K][N] row-major with an exact power-of-two scale
 * 2^t chosen so max|B| maps near 2^14; t is added to *d_exp (may be NULL: t = 0);
 * *d_b_bound receives max column 1-norm of the stored B_P (float).  Two kernels. */
TN_API int tn_pad_b(void* d_bp, const void* d_b, uint32_t K, uint32_t N, float* d_b_bound, int* d_exp,
             void* d_scratch /* >= 16 bytes */, void* stream);

/* Eq. 1 int8 group codec on a flat fp32 array (g reals per group, exp = 1, reading C-A10..C-A13):
 * codes int8, scales/zeros fp32 per group. n must be a multiple of g. */
TN_API int tn_quant_int8(int8_t* d_codes, float* d_scales, float* d_zeros, const float* d_x, uint64_t n,
                  int g, void* stream);
TN_API int tn_dequant_int8(float* d_y, const int8_t* d_codes, const float* d_scales, const float* d_zeros,
                    uint64_t n, int g, void* stream);
/* Fused sender side of a quantised mode swap (north_star (5); Alg. 1 P:357-361 + Eq. 1
 * P:389-406): the codec applied to Y = X.transpose(perm) without materialising Y.  X is a
 * complex-half tensor of rank n (all dims 2, interleaved fp16 re/im, 2^(n+1) reals), perm follows
 * tn_permute (output axis j = input axis perm[j], axis 0 outermost).  codec TN_COMM_INT8 writes
 * 2^(n+1) int8 codes, TN_COMM_INT4 2^n packed bytes (tn_quant_int4_f16 layout); scales/zeros get
 * 2^(n+1)/g floats.  Codes/scales/zeros are bit-identical to tn_permute then tn_quant_*_f16.
 * Requires g a power of two >= 2 and perm keeping the innermost log2(g/2) axes in place
 * (else TN_E_INVALID, nothing launched).  Device pointers; X must not alias the outputs. */
TN_API int tn_permute_quant_f16(void* d_codes, float* d_scales, float* d_zeros, const void* d_x, int n,
                                const int* perm, int g, int codec, void* stream);
/* Same codec on fp16 reals (the complex-half mode-swap payload): the codec's input is the exact
 * float32 value of each fp16; dequantised values are rounded to fp16 (round to nearest even). */
TN_API int tn_quant_int8_f16(int8_t* d_codes, float* d_scales, float* d_zeros, const void* d_x, uint64_t n,
                             int g, void* stream);
TN_API int tn_dequant_int8_f16(void* d_y, const int8_t* d_codes, const float* d_scales, const float* d_zeros,
                               uint64_t n, int g, void* stream);
/* Table 1 int8 preset codec with exponent (Eq. 1 with exp, reading C-A10) on fp16 reals, groups of g
 * reals (g a power of two dividing n; the mode swap uses g = one destination chunk, e = 0.2):
 * x' = sign(x)|x|^e (double pow, rounded to fp32), scale/zero of Eq. 1 from max/min of x' per group,
 * code = rint(x' scale + zero) clamped to [-128, 127] (fp32 multiply then add); dequantised
 * y = sign(y')|y'|^(1/e), y' = (code - zero)/scale, rounded to fp16.  Constant groups: scale 0, zero =
 * the transformed constant.  d_tmp: device scratch of 8 * n/g bytes.  Two/one kernels. */
TN_API int tn_quant_int8_exp_f16(int8_t* d_codes, float* d_scales, float* d_zeros, const void* d_x, uint64_t n,
                                 uint64_t g, double e, void* d_tmp, void* stream);
TN_API int tn_dequant_int8_exp_f16(void* d_y, const int8_t* d_codes, const float* d_scales, const float* d_zeros,
                                   uint64_t n, uint64_t g, double e, void* stream);
/* int4 preset (Table 1: q in [0, 15], exp 1, groups of g reals) on fp16
 * reals: n/2 packed bytes, two codes per byte with the low nibble = even index (reading C-A14);
 * scale = 15/(max-min), zero = -15*min/(max-min) per group (fp32, multiply then add, no FMA;
 * constant groups: scale 0, zero = the constant, codes 0).  g even, n a multiple of g. */
TN_API int tn_quant_int4_f16(uint8_t* d_packed, float* d_scales, float* d_zeros, const void* d_x, uint64_t n,
                             int g, void* stream);
TN_API int tn_dequant_int4_f16(void* d_y, const uint8_t* d_packed, const float* d_scales, const float* d_zeros,
                               uint64_t n, int g, void* stream);

/* ---- multi-GPU (stem sharded on its log2(world) outermost modes, Alg. 1) ---- */
TN_API int tn_comm_unique_id(uint8_t out[128]);
TN_API int tn_comm_init(const uint8_t uid[128], int rank, int world, int device, tn_comm** out);
/* Loopback transport (testing and schedule validation on one GPU): `world` virtual ranks that all
 * live on `device`.  out[r] (caller array of `world` pointers) receives rank r's communicator; each
 * is passed to its own tn_plan_load and freed with tn_comm_free.  Every collective of the sharded
 * path (mode-swap exchanges, the per-step max all-reduce, the readout all-gather) becomes a host
 * rendezvous of the virtual ranks plus device-to-device copies ordered by CUDA events, so the same
 * lowering, codec kernels and swap schedule run as with NCCL.  Each virtual rank's plan must be
 * driven from its OWN host thread (a rendezvous blocks until every rank arrives; it fails with
 * TN_E_NCCL after 600 s).  Each rank needs its own buffers; the stem shards are 1/world of the stem,
 * so world virtual ranks fit wherever one rank holding the whole stem fits. */
TN_API int tn_comm_init_loopback(int world, int device, tn_comm** out);
TN_API void tn_comm_free(tn_comm* c);

#ifdef __cplusplus
}
#endif
#endif /* TN_H_ */
