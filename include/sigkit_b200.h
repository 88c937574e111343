/*
 * sigkit_b200.h -- C ABI of the B200-native word-basis signature engine.
 *
 * This is the drop-in seam for the reference package `sigkit` (paths relative
 * to /root/reference/pkg/src/sigkit).  The reference crosses from Python into
 * compiled code at exactly three call sites, all numba kernels that receive
 * caller-allocated C-contiguous arrays and return nothing:
 *
 *   sigcore.py:238   _kernels.forward_kernel(incr, letters, lengths, inv, out)
 *   sigcore.py:258   _kernels.windows_kernel(incr, letters, lengths, bounds, inv, out)
 *   backward.py:203  _kernels.backward_kernel(incr, letters, lengths, upstream, inv,
 *                                            stride, left, right, dh, acc, ckpt, inc_grads)
 *
 * plus the word-set tables those kernels consume (wordsets.py:176-247).  The
 * functions below replace them one for one (see each comment).  Conventions:
 *
 *   - every pointer named d_* is DEVICE memory owned by the caller; the
 *     library never allocates persistent device memory except inside a plan;
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it;
 *   - every function returns SIGB_OK (0) or one of the SIGB_ERR_* codes below,
 *     which the Python layer maps onto the reference's SigkitError hierarchy
 *     (errors.py:4-37); sigb_last_error() returns the message (thread-local);
 *   - dtype is SIGB_F32 or SIGB_F64, the dtype of samples/outputs;
 *   - results are deterministic: no floating-point atomics anywhere, every
 *     reduction runs in a fixed order (the reference's bitwise
 *     thread-count-invariance contract, _kernels.py:5-7).
 */
#ifndef SIGKIT_B200_H
#define SIGKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIGB_OK 0
#define SIGB_ERR_SHAPE 1       /* ShapeError      (errors.py:26) */
#define SIGB_ERR_DOMAIN 2      /* DomainError     (errors.py:22) */
#define SIGB_ERR_CAPACITY 3    /* CapacityError   (errors.py:10) */
#define SIGB_ERR_UNSUPPORTED 4 /* UnsupportedWordSetError (errors.py:34) */
#define SIGB_ERR_CUDA 5        /* device / launch failure */

#define SIGB_F32 0
#define SIGB_F64 1

/* ABI version (major * 100 + minor). */
int sigb_version(void);
/* Message of the last failing call on this host thread. */
const char* sigb_last_error(void);
/* Number of SMs of the current device (grid sizing helper). */
int sigb_device_sm_count(void);
/* Kernel routing: 0 = auto (register-resident truncated kernels where an
 * instantiation exists, else fragment kernels, else level kernels),
 * 1 = level kernels only, 2 = fragment kernels (then level kernels),
 * 4 = word-set-specialised generated kernels (then fragment, level kernels).
 * Process-wide; used by the tests to check both paths against the oracle.
 * (Policy 3, the round-1 level-slot kernels, was removed and is rejected.) */
int sigb_set_kernel_policy(int policy);
/* Tensor-core precision contract for float32 full truncations with d = 16, depth 4
 * (config 5 shape).  on = 1 (default): the forward's leaf level runs as 3xTF32 on
 * tcgen05 (hi/lo split of both operands, fp32 accumulation; measured <= 3.4e-6
 * relative on S at c5) and the backward's two leaf sums as a scaled 3-pass fp16 split
 * (power-of-two row / column scales, fp32 accumulation; <= 1.3e-6 relative on dL/dX),
 * both well inside the 1e-4 float32 gate.  on = 0: the CUDA-core fp32 kernels
 * (bitwise-reproducible against each other, ~15-60% slower).  float64 never uses
 * the tensor cores.  Process-wide; the environment variables SIGB_TRUNC_TC=0 /
 * SIGB_TRUNC_TC_BWD=0 select the CUDA-core kernels as well.  Returns the previous
 * setting.  No reference counterpart (the reference is CPU-only, fp64 backward). */
int sigb_set_tensor_cores(int on);
/* Number of device kernels this library has launched (process-wide). */
long long sigb_launch_count(void);
/* CUDA-event timing of the main Chen kernels, recorded on the launch stream
 * (bench.py's roofline leg).  sigb_timing_enable(1) resets and arms it;
 * sigb_timing_read(which, &ms, &n) synchronises on the recorded events and
 * returns the summed device time and launch count since the last read,
 * which = 0 forward kernel, 1 backward kernel.  No reference counterpart
 * (the reference times whole calls with perf_counter, bench.py:25-39). */
int sigb_timing_enable(int on);
int sigb_timing_read(int which, double* ms, int64_t* launches);

/*
 * Word-set tables on device.  Replaces WordSet.letters (wordsets.py:176-188),
 * WordSet.prefix_table / suffix_table (wordsets.py:190-228, sentinels
 * EPSILON_INDEX=-1, MISSING_INDEX=-2 at wordsets.py:31-34), the level
 * offsets behind _level_counts/_level_start/level_slice (wordsets.py:230-247)
 * and pack_letters (words.py:158-174).  Input: the canonical (length asc,
 * code asc) arrays WordSet.lengths / WordSet.codes.  Bit-exact with the
 * reference.  d_packed may be NULL (it needs bits_per_letter*max_len <= 64).
 *   d_letters     int64 (W, max_len)
 *   d_prefix      int64 (W, max_len + 1)
 *   d_suffix      int64 (W, max_len + 1)
 *   d_level_start int64 (max_len + 2): start of level n at [n], total at [max_len+1]
 *   d_packed      uint64 (W)
 */
int sigb_wordset_tables(const uint64_t* d_codes, const int64_t* d_lengths, int64_t W, int64_t d,
                        int64_t max_len, int64_t* d_letters, int64_t* d_prefix, int64_t* d_suffix,
                        int64_t* d_level_start, uint64_t* d_packed, void* stream);

/*
 * Execution plan of one word set (opaque).  Built from the host copies of
 * WordSet.codes / WordSet.lengths: computes the prefix closure cl(I) (the
 * reference computes missing prefixes as scratch, wordsets.py:8-9), runs
 * sigb_wordset_tables on it, and derives the kernels' schedule (parent /
 * child / level tables, partition of the trie into independent parts).
 * Holds device memory until sigb_plan_destroy.  The plan belongs to the device
 * current at sigb_plan_create; every call taking the plan makes that device
 * current for its duration (and restores the caller's), so buffers and stream
 * must live on it.
 */
typedef struct sigb_plan sigb_plan;

int sigb_plan_create(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d,
                     sigb_plan** plan, void* stream);
int sigb_plan_destroy(sigb_plan* plan);
/* |cl(I)| -- width of the closure state used by sigb_backward when I is not prefix-closed. */
int64_t sigb_plan_closure_size(const sigb_plan* plan);
/* Number of independent trie parts (diagnostics / DESIGN.md). */
int64_t sigb_plan_num_parts(const sigb_plan* plan);
/* Executed FMA count of one Chen step of one path (T-node count; diagnostics). */
int64_t sigb_plan_step_fmas(const sigb_plan* plan);
/* Thread blocks the forward launches for B whole paths on this plan's register-resident
 * truncated kernels (-1 for other kernel families): the host side's fill measure for the
 * parallel-in-time route of small batches (signature.py _scan_forward). */
int64_t sigb_forward_ctas(const sigb_plan* plan, int64_t B);
/* Kernel family sigb_forward / sigb_backward will run for this plan under the
 * current policy: 1 = register-resident truncated kernels, 2 = register-resident
 * fragment kernels (any trie), 4 = word-set-specialised generated kernels (small sparse sets),
 * 0 = level-synchronous trie kernels, -1 = NULL plan. */
int sigb_plan_kernel_kind(const sigb_plan* plan);
/* Host-only (no device): the fragment decomposition the plan would use for
 * this word set.  info[8] = {NC, G, K, fragments, CTAs per path, |cl(I)|,
 * estimated issue slots per path-step, instantiated (0/1)}.  Fails with
 * SIGB_ERR_UNSUPPORTED when no fragment shape fits. */
int sigb_fragment_plan_info(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d, int64_t* info);
/* Host-only: the CUDA source generated for a small word set (the plan
 * compiles it with NVRTC for sm_100a on first use; policy 4 / auto for sparse
 * sets).  Writes at most cap-1 bytes + NUL to buf (may be NULL) and the full
 * length to *len.  SIGB_ERR_UNSUPPORTED when the set is too large. */
int sigb_jit_source(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d, int dtype, int backward,
                    char* buf, size_t cap, size_t* len);
/* Host-only: generate and NVRTC-compile the set's kernel for sm_100a into the
 * cubin cache (jit_cache/ next to the library, or $SIGB_JIT_CACHE), so a
 * device process loads it instead of compiling on first use.  The build runs
 * it for the shipped word sets (config 3). */
int sigb_jit_precompile(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d, int dtype, int backward);

/*
 * Forward signature.  Replaces forward_kernel (_kernels.py:40-58) together
 * with the increments (sigcore.py:80-88, fused: the kernel differences the
 * samples itself) and the epsilon column (sigcore.py:218-224).
 *   d_X      (B, L, d) samples, dtype
 *   d_out    row b at d_out + b*out_ld; word k of I is written at column out_col0+k;
 *            if include_empty, column out_col0-1 is set to 1 (needs out_col0 >= 1)
 *   d_state  NULL, or (B, |cl(I)|) terminal closure state (needed by sigb_backward
 *            when I is not prefix-closed)
 * L == 1 (no increments) yields the identity (zeros), as the reference.
 */
int sigb_forward(const sigb_plan* plan, int dtype, const void* d_X, int64_t B, int64_t L,
                 void* d_out, int64_t out_ld, int64_t out_col0, int include_empty, void* d_state,
                 void* stream);

/*
 * Windowed signatures.  Replaces windows_kernel (_kernels.py:61-82):
 * d_bounds int64 (K, 2) sample-index pairs 0 <= l < r <= L-1 (validated by
 * the caller, sigcore.py:138-163); d_out (B, K, W) -- window k of path b
 * at d_out + (b*K + k)*W.
 */
int sigb_windows(const sigb_plan* plan, int dtype, const void* d_X, int64_t B, int64_t L,
                 const int64_t* d_bounds, int64_t K, void* d_out, void* stream);

/*
 * Backward.  Replaces backward_kernel (_kernels.py:85-183) fused with
 * increment_to_sample_grads (backward.py:130-147).  Memory-lean: consumes
 * the terminal signature instead of a stored trajectory and rebuilds
 * S_{0,t_j} by multiplying with exp(-dX_j) while sweeping j = M-1..0.
 *   d_S      terminal state: (B, W) forward output (out_ld/out_col0 layout of
 *            sigb_forward) when I is prefix-closed, else the d_state (B, |cl(I)|)
 *            of sigb_forward (set s_is_state = 1)
 *   d_g      upstream dL/dS, row b at d_g + b*g_ld, word k at column g_col0 + k
 *            (a leading epsilon column is skipped by passing g_col0 = 1,
 *            backward.py:177-178)
 *   ckpt_stride  0 = pure reconstruction; c > 0 = reload exact S_{0,t_j}
 *            every c steps from checkpoints taken by a forward replay
 *            (the reference's accuracy dial, backward.py:183-199)
 *   d_work   workspace of sigb_backward_workspace_size bytes
 *   d_dX     (B, L, d) dL/dX, dtype (the path gradients, fully overwritten)
 *   d_dinc   NULL or (B, L-1, d) dL/d(dX_j) (GradBatch.increment_grads)
 */
int sigb_backward_workspace_size(const sigb_plan* plan, int dtype, int64_t B, int64_t L,
                                 int64_t ckpt_stride, size_t* bytes);
int sigb_backward(const sigb_plan* plan, int dtype, const void* d_X, int64_t B, int64_t L,
                  const void* d_S, int64_t s_ld, int64_t s_col0, int s_is_state, const void* d_g,
                  int64_t g_ld, int64_t g_col0, int64_t ckpt_stride, void* d_work, size_t work_bytes,
                  void* d_dX, void* d_dinc, void* stream);

/*
 * Log-signature polynomial (the consumers of signature_forward that
 * logsig.py routes through the hot path).  Replaces the numpy loops of
 * logsignature_forward (logsig.py:165-173) and logsignature_backward
 * (logsig.py:208-222) over the host-built term table of _lyndon_projection
 * (logsig.py:79-127): Lyndon word i has terms [term_off[i], term_off[i+1]);
 * term t is coef[t] * prod_k sig[cols[t*F + k]] over its factor columns
 * (F = max_factors, -1 padded), coef = (-1)^(k+1)/k for k factors.
 *   forward:  out[b*out_ld + i] = sum_t coef[t] prod_k sig[b*sig_ld + cols[t][k]]
 *   backward: up[b*up_ld + c] = sum over entries e of column c, e = (t << 8) | k,
 *             of g[b*g_ld + term_word[t]] * coef[t] * prod_{k' != k} sig[..cols[t][k']]
 *             (the column -> (term, factor) index replaces the reference's
 *             scatter-add, so the sum runs in a fixed order).
 */
int sigb_logsig_forward(int dtype, const void* d_sig, int64_t B, int64_t sig_ld, const int64_t* d_term_off,
                        const int32_t* d_cols, const double* d_coef, int64_t n_out, int max_factors, void* d_out,
                        int64_t out_ld, void* stream);
int sigb_logsig_backward(int dtype, const void* d_sig, int64_t B, int64_t sig_ld, const void* d_g, int64_t g_ld,
                         const int64_t* d_col_off, const int64_t* d_entries, const int64_t* d_term_word,
                         const int32_t* d_cols, const double* d_coef, int max_factors, int64_t ncols, void* d_up,
                         int64_t up_ld, void* stream);
/*
 * Graded product of dense truncated tensors in the epsilon-first layout
 * (width sum_{n<=N} d^n, row b at b*width): replaces _tensor_mul_full
 * (sigcore.py:297-311), the kernel of chen_concat (sigcore.py:321-334),
 * signature_inverse (sigcore.py:337-352), tensor_log and tensor_exp
 * (logsig.py:42-72):  out = scale * (x (x) y), then out[:, 0] += add0.
 * d_out must not alias d_x or d_y.
 */
int sigb_tensor_mul(int dtype, const void* d_x, const void* d_y, int64_t B, int64_t d, int N, double scale,
                    double add0, void* d_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SIGKIT_B200_H */
