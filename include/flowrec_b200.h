/* C ABI of the B200 jet-MLP training engine (libflowrec_b200.so).
 *
 * This is the drop-in boundary for the reference's training hot path
 * (arXiv 2602.15883, package `flowrec`).  Every entry point is asynchronous on
 * the caller's CUDA stream, takes caller-owned device buffers (plain pointers
 * and sizes), performs no allocation (so every call is CUDA-graph capturable)
 * and returns 0 on success or a non-zero status with a message available from
 * fr_last_error().
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/flowrec):
 *   fr_plan_create        autodiff/builders.py:14-21,67-100 (_validate_arch, tape build)
 *                         + tape.py:298-326 (per-bind shape checks, now done once)
 *   fr_prepare_params     tape.py:314-326 (Tape.bind_params: params bound by reference)
 *   fr_pde_fwd_bwd        builders.py:85-100 build_pde_tape + tape.py:329-371 fwd/bwd
 *   fr_mse_fwd_bwd        builders.py:103-141 build_mse_tape + tape.py:329-371
 *   fr_epoch_fwd_bwd      runtime/objective.py:164-182 (all of one rank's loss heads)
 *   fr_value_fwd          builders.py:67-73 build_value_tape; network.py:142-156 predict
 *   fr_jet_fwd            builders.py:76-82,192-203 build_jet_tape/forward_jet;
 *                         network.py:162-177 predict_jet
 *   fr_reduce_grad        tape.py:365-371 (adjoint scatter into the flat grad, W0,b0,...)
 *   fr_reduce_loss        objective.py:46-64 (_MiniBatched.run scalar sums)
 *   fr_adam_step          runtime/optim.py:20-49 (clip_by_global_norm + adam_step),
 *                         objective.py:183-198 (LossParts, compose_loss, finiteness),
 *                         worker.py:231-244 (run_epoch history row)
 *   fr_pack_ghost         runtime/worker.py:24-46,170-198 (anchor_normalize, messages)
 *   fr_jet_act_forward    _kernels/__init__.py:57-60 jet_act_forward  (_cyjet.pyx:11-34)
 *   fr_jet_act_backward   _kernels/__init__.py:63-68 jet_act_backward (_cyjet.pyx:37-86)
 */
#ifndef FLOWREC_B200_H
#define FLOWREC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fr_stream_t; /* == cudaStream_t */
typedef struct fr_plan fr_plan;

enum { FR_ACT_TANH = 0, FR_ACT_SIN = 1 };                                /* _kernels ACT_* */
enum { FR_STEADY2D = 0, FR_UNSTEADY2D = 1, FR_UNSTEADY3D = 2 };          /* physics._KINDS */
enum { FR_F32 = 0, FR_F64 = 1 };
enum { FR_MODE_PDE = 0, FR_MODE_MSE = 1, FR_MODE_VALUE = 2, FR_MODE_JET = 3, FR_MODE_GJ = 4 };
enum { FR_FLAG_NONFINITE_LOSS = 1, FR_FLAG_NONFINITE_GRAD = 2, FR_FLAG_EXCHANGE_TIMEOUT = 4 };
/* contraction math of the training kernels: FP32 SIMT (oracle parity ~1e-5) or
 * TF32 tcgen05 tensor cores (wide FP32 experts, 64 < width <= 512; default) */
enum { FR_MATH_SIMT = 0, FR_MATH_TF32 = 1, FR_MATH_TF32X3 = 2 };
/* FR_MATH_TF32X3: the W <= 64 fused epoch kernel's forward and adjoint hidden
 * contractions on tcgen05 as split TF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi,
 * FP32 accumulation in TMEM; ~FP32 accuracy) */

typedef struct {
  int n_in, n_out, n_vel, hidden_layers, width, width_pad;
  int n_params;      /* reference flat parameter count (network.py:112-115) */
  int np_pad;        /* kernel gradient-partial row length */
  int kp_elems;      /* elements of the prepared kernel-parameter buffer */
  int dtype, act, regime, num_sms;
  double inv_re;
  int math;          /* FR_MATH_* of the PDE / MSE training kernels */
  int tc_width;      /* hidden width of the TF32 tcgen05 kernels (rounded to 16 / 32; 0: none) */
} fr_plan_info;

typedef struct {
  int grid;           /* CTAs == gradient / loss partial rows written */
  int threads;        /* threads per CTA */
  int points_per_tile;
  int jet_streams;    /* rows per point in JET mode output (n, S, n_out) */
  long long gpart_elems;   /* doubles: grid * np_pad (0 for forward-only modes) */
  long long lpart_elems;   /* doubles: grid * 2 */
  long long scratch_bytes; /* per-call stash workspace */
  size_t smem_bytes;
  int loss_rows;           /* rows of 2 doubles in lpart (== grid for the fused kernels) */
  int wide;                /* 1: layer-wise SIMT wide kernels (hidden width > 64), 2: TF32 tcgen05 wide kernels */
  long long tiles;         /* work tiles of the launch (persistent kernels deal them round robin) */
} fr_workspace;

/* Plan: validated network + regime description (replaces per-bind checks). */
int fr_plan_create(const int* arch, int n_arch, int act, int regime, double inv_re, int dtype,
                   fr_plan** out);
int fr_plan_destroy(fr_plan* plan);
int fr_plan_get_info(const fr_plan* plan, fr_plan_info* out);
/* select FR_MATH_SIMT, FR_MATH_TF32 (wide experts) or FR_MATH_TF32X3 (the W <= 64
 * fused epoch kernel) for the plan's training kernels */
int fr_plan_set_math(fr_plan* plan, int math);
int fr_plan_workspace(const fr_plan* plan, int mode, long long n, fr_workspace* out);

/* flat f64 params (reference layout) -> padded kernel params (+ W^T copies) */
int fr_prepare_params(const fr_plan* plan, const double* flat, void* kparams, fr_stream_t stream);

/* PDE residual loss over n collocation points: per-CTA f64 gradient partials of
 * coef * sum_n |r_n|^2 and per-CTA f64 sums of |r_n|^2 (lpart[2*cta]). */
int fr_pde_fwd_bwd(const fr_plan* plan, const void* kparams, const void* pts, long long n,
                   double coef, double* gpart, double* lpart, void* scratch, fr_stream_t stream);

/* MSE head: vel_coef * sum_n sum_c w_c (u_c - tu_c)^2 + p_coef * sum_n (p - tp)^2;
 * target_p == NULL omits the pressure term (builders.py:133-139). */
int fr_mse_fwd_bwd(const fr_plan* plan, const void* kparams, const void* pts, const void* target_u,
                   const void* target_p, long long n, const double* vel_w, double vel_coef,
                   double p_coef, double* gpart, double* lpart, void* scratch, fr_stream_t stream);

/* One launch for a whole epoch's loss heads: the PDE residual over the
 * collocation points plus up to three MSE sets (obs, ghost-spatial,
 * ghost-temporal; target_p NULL omits a set's pressure term).  Every CTA adds
 * all its contributions into one f64 gradient-partial row (gpart: grid rows of
 * np_pad); loss partials go to per-set blocks of `grid` rows x 2 in lpart:
 * lpart_blocks[0] <- the PDE, lpart_blocks[1 + s] <- set s. */
typedef struct {
  const void* pts;
  const void* target_u;
  const void* target_p;
  long long n;
  double vel_coef;
  double p_coef;
} fr_mse_set;

int fr_epoch_workspace(const fr_plan* plan, long long n_colloc, const long long* n_sets, int n_set_count,
                       fr_workspace* out);
int fr_epoch_fwd_bwd(const fr_plan* plan, const void* kparams, const void* colloc, long long n_colloc,
                     double pde_coef, const fr_mse_set* sets, int n_set_count, const double* vel_w,
                     double* gpart, double* const* lpart_blocks, void* scratch, fr_stream_t stream);

/* Ghost-exchange overlap (worker.py:170-228 / driver.py:133-142).
 * The epoch launch starts before this rank's ghost targets have arrived: the
 * MSE sets from `first_gated_set` on (the ghost sets; obs is never gated) wait
 * inside the kernel until *gate != 0, which the transport stream sets with
 * fr_signal() once the NCCL receives (or in-process copies) have landed.  Each
 * CTA reaches its ghost tiles only after all of its PDE and obs tiles, so the
 * exchange latency hides under the interior work.  max_ctas caps the SMs the
 * persistent grid may occupy (its CTAs = that many SMs x CTAs per SM), so the
 * transport's kernels keep free SMs (0 = every SM); the workspace
 * must be sized with the same cap (fr_epoch_workspace_capped).  A wait longer
 * than timeout_ms or-s FR_FLAG_EXCHANGE_TIMEOUT into *flags and proceeds (the
 * host raises; drop-in for the reference's DeadlockError, driver.py:161-166). */
typedef struct {
  const unsigned* gate;
  int first_gated_set;
  int max_ctas;
  int* flags;
  unsigned timeout_ms;
  /* peer-memory transport: when gate_round is non-NULL the gate is a monotonic
   * arrival counter and the ghost sets wait until *gate >= *gate_round * gate_mult
   * (gate_mult = incoming edges per round; *gate_round = rounds so far) */
  const unsigned* gate_round;
  unsigned gate_mult;
} fr_epoch_gate;

/* gate == NULL, or a gate whose `gate` word is NULL: nothing waits; the latter
 * still applies max_ctas (ungated epochs of a trainer whose workspace was sized
 * with a cap must launch the same grid). */
int fr_epoch_workspace_capped(const fr_plan* plan, long long n_colloc, const long long* n_sets, int n_set_count,
                              int max_ctas, fr_workspace* out);
int fr_epoch_fwd_bwd_gated(const fr_plan* plan, const void* kparams, const void* colloc, long long n_colloc,
                           double pde_coef, const fr_mse_set* sets, int n_set_count, const double* vel_w,
                           double* gpart, double* const* lpart_blocks, void* scratch, const fr_epoch_gate* gate,
                           fr_stream_t stream);
/* *word = value once every prior operation on `stream` has completed (one
 * single-thread kernel, release ordering); with delay_ns > 0 it first sleeps
 * that long on the device (tests emulate a slow transport with it) */
int fr_signal(unsigned* word, unsigned value, unsigned delay_ns, fr_stream_t stream);

/* Ghost-derivative matching (opt-in extension of the reference's value-only
 * coupling, worker.py:179-197): loss sum_n sum_i sum_c
 * w_c (d u_c / d x_i (pts_n) - target_du[n][i][c])^2 over the first
 * derivatives of the velocity w.r.t. every input, times coef in the gradient;
 * gpart / lpart / scratch as for fr_pde_fwd_bwd (workspace of FR_MODE_GJ). */
int fr_ghost_jet_fwd_bwd(const fr_plan* plan, const void* kparams, const void* pts, const void* target_du,
                         long long n, const double* vel_w, double coef, double* gpart, double* lpart, void* scratch,
                         fr_stream_t stream);

/* Ghost-exchange transport over NCCL point-to-point.  libnccl.so.2
 * is resolved at run time (the copy a PyTorch process already holds).
 * fr_nccl_get_unique_id writes 128 bytes on one rank; every rank passes them
 * to fr_nccl_init.  fr_exchange enqueues one grouped round -- all sends and
 * receives of this rank -- on `stream`; counts are elements of `dtype`
 * (FR_F32 / FR_F64). */
typedef struct fr_comm fr_comm;
int fr_nccl_get_unique_id(void* id_out);
int fr_nccl_init(const void* unique_id, int nranks, int rank, fr_comm** out);
int fr_nccl_destroy(fr_comm* comm);
int fr_exchange(fr_comm* comm, int n_send, const int* send_peers, const void* const* send_bufs,
                const long long* send_counts, int n_recv, const int* recv_peers, void* const* recv_bufs,
                const long long* recv_counts, int dtype, fr_stream_t stream);

/* Peer-memory ghost transport (one process per GPU over NVLink / NVSwitch, or
 * several ranks in one process).  Each rank allocates its ghost-target rows and
 * its sync words in one block with fr_ipc_alloc (cudaMalloc + IPC handle of 64
 * bytes); peers map it with fr_ipc_open (peer access enabled lazily).  The
 * producer's pack then stores straight into the destination's target rows --
 * no staging buffer, no NCCL kernel -- so the whole epoch (producer -> put ->
 * gated epoch kernel -> reductions -> Adam) is one CUDA graph.
 *
 * Sync words per rank (u32, monotonic, zero-initialised):
 *   ready    -- + 1 by every source after its rows for this rank landed
 *               (release, system scope); the epoch kernel's ghost sets wait
 *               for ready >= rounds * n_incoming (fr_epoch_gate.gate_round)
 *   epochs   -- + 1 by the rank itself after each epoch kernel (its targets
 *               are free again); a source writes round k's rows for an epoch e
 *               only once the destination's `epochs` has reached e (WAR guard),
 *               comparing against its own `epochs` word (ranks run the same
 *               epoch sequence) */
typedef struct {
  long long y_row;          /* first row of this edge in the producer's value output y */
  long long anchor_row;     /* rows of the anchor evaluations (masters), or -1 */
  long long n;              /* ghost points */
  void* u;                  /* destination's target rows (n, n_vel), peer pointer */
  void* p;                  /* (n,) */
  void* du;                 /* (n, n_in, n_vel) derivative targets or NULL (C^1 extension) */
  unsigned* ready;          /* destination's ready word (peer pointer) */
  const unsigned* epochs;   /* destination's epochs word (peer pointer) */
} fr_ghost_edge;
#define FR_MAX_GHOST_EDGES 16

int fr_ipc_alloc(size_t bytes, void** ptr, void* handle_out);
int fr_ipc_open(const void* handle, void** ptr);
int fr_ipc_close(void* ptr);
int fr_ipc_free(void* ptr);
/* One round of this rank's outgoing edges: per edge wait (bounded by timeout_ms;
 * FR_FLAG_EXCHANGE_TIMEOUT into *flags) until *edge.epochs >= *my_epochs, store
 * u = y[:, :n_vel], p = y[:, p] - y_anchor[:, p] (anchor-normalised on masters,
 * worker.py:24-46,170-198) [and du from y_jet (n, 1 + 2 n_in, n_out)] into the
 * destination, then release-add 1 to *edge.ready. */
int fr_ghost_put(const fr_plan* plan, const void* y, const void* y_jet, int n_edges, const fr_ghost_edge* edges,
                 const unsigned* my_epochs, unsigned timeout_ms, int* flags, fr_stream_t stream);
/* *word += value (release, system scope) once prior work on `stream` is done */
int fr_counter_add(unsigned* word, unsigned value, fr_stream_t stream);

/* GPU-side dataset sampling: out[i][j] (row-major n x n_cols,
 * f64 and/or f32) = the value NumPy's Generator(PCG64) produces for
 * rng.uniform(lo[j], hi[j], size=n) called once per column j in order
 * (decomposition.py:64-70), starting `skip` draws into the stream whose state
 * before the first draw is state4 = {state >> 64, state & (2^64-1), inc >> 64,
 * inc & (2^64-1)} (e.g. PCG64(SeedSequence([seed, rank, tag])).state).  Bit-exact. */
int fr_pcg64_uniform(const unsigned long long* state4, unsigned long long skip, long long n, int n_cols,
                     const double* lo, const double* hi, double* out64, float* out32, fr_stream_t stream);

/* value forward: out (n, n_out) */
int fr_value_fwd(const fr_plan* plan, const void* kparams, const void* pts, long long n, void* out,
                 fr_stream_t stream);
/* jet forward: out (n, 1 + 2*n_in, n_out): value, d/dx_j, d2/dx_j^2 */
int fr_jet_fwd(const fr_plan* plan, const void* kparams, const void* pts, long long n, void* out,
               fr_stream_t stream);

/* grad[i] (+)= sum_rows gpart[row][pad(i)], fixed row order; when norm_parts is
 * non-NULL also writes per-block partial sums of grad^2 (fr_reduce_grad_parts()
 * entries) for fr_adam_step */
int fr_reduce_grad(const fr_plan* plan, const double* gpart, int rows, double* grad, int accumulate,
                   double* norm_parts, fr_stream_t stream);
int fr_reduce_grad_parts(const fr_plan* plan);
/* sums[2*s + c] = sum over rows of segment s of lpart[2*row + c], fixed order */
int fr_reduce_loss(const double* lpart, const int* seg_rows_host, int n_seg, double* sums,
                   fr_stream_t stream);

typedef struct {
  /* optimiser state (device, f64, length n) */
  long long n;
  double* params;
  double* grad;
  double* m;
  double* v;
  long long* step;          /* device counter, AdamState.step */
  /* schedule: row r = *step - row_base holds {lr, 1 - beta1^t, 1 - beta2^t} for
   * t = *step + 1 (host-computed, bit-identical to the reference's Python float
   * math); history and grad_norm rows use the same index r */
  const double* sched;
  long long row_base;
  double beta1, beta2, eps, clip_norm; /* NaN: no clipping (the reference's None); otherwise
                                        the gradient is scaled by clip_norm / norm whenever
                                        norm > clip_norm (optim.py:26-27) */
  /* squared-norm partials written by fr_reduce_grad (NULL: reduce grad here) */
  const double* norm_parts;
  int n_norm_parts;
  /* loss bookkeeping (lpart == NULL -> no history / finiteness check): per-CTA
   * loss partial rows of the datasets {obs, pde, ghost-spatial, ghost-temporal},
   * seg_rows[s] rows each, contiguous in that order */
  const double* lpart;
  int seg_rows[4];
  double n_obs, n_colloc, n_ghost_total, n_ghost_space, n_ghost_time;
  double w_obs, w_pde, w_ghost_u, w_ghost_p_space, w_ghost_p_time;
  double* history;          /* rows of 7: epoch, 5 unweighted parts, lr */
  int* flags;               /* FR_FLAG_* bits, sticky */
  double* grad_norm;        /* optional: pre-clip norm per step (row index) */
  void* kparams;            /* optional: refresh prepared kernel params */
  int* sync_counter;        /* device int, zero-initialised, self-resetting */
} fr_adam_args;

/* plan may be NULL when kparams is NULL (plain flat-vector Adam) */
int fr_adam_step(const fr_plan* plan, const fr_adam_args* args, fr_stream_t stream);

/* ghost message: u = y[:, :n_vel]; p = y[:, p] - (y_anchor ? y_anchor[:, p] : 0) */
int fr_pack_ghost(const fr_plan* plan, const void* y, const void* y_anchor, long long n, void* out_u,
                  void* out_p, fr_stream_t stream);

/* The reference's native seam (f64, stacked layout ((1+2d)*batch, width)). */
int fr_jet_act_forward(int kind, const double* z, double* s, const double* aux, double* d1,
                       double* d2, long long batch, int n_inputs, int width, fr_stream_t stream);
int fr_jet_act_backward(int kind, const double* z, const double* s, const double* aux,
                        const double* sbar, double* zbar, long long batch, int n_inputs, int width,
                        int accumulate, fr_stream_t stream);

/* FP32 FFMA throughput probe (measured SIMT roofline denominator): grid x 256
 * threads, each running `iters` x 64 independent FMA chains of 8; out[grid*256] */
int fr_bench_ffma(int grid, int iters, int unused, float* out, fr_stream_t stream);

/* tcgen05 probe: C[128][N] = A[128][K] * B[N][K]^T in TF32 on the tensor core,
 * accumulator in TMEM (16 <= N <= 256, N % 16 == 0, K % 8 == 0, K <= 64);
 * layout bit 0 / bit 1 stage A / B MN-major instead of K-major */
int fr_debug_tc_gemm_tf32(const float* A, const float* B, float* C, int N, int K, int layout, fr_stream_t stream);
/* tcgen05 layout discovery: C[128][32] = words of A's shared tile (filled with
 * their own indices) that one 128x32xK MMA reads under descriptor (lbo, sbo) */
int fr_debug_tc_raw(float* C, int K, int a_mn, int lbo, int sbo, fr_stream_t stream);
int fr_debug_tc_raw2(float* C, int a_mn, int lbo, int sbo, int ltype, int shift, fr_stream_t stream);
/* TMA view probe: one 32-row group of a k-quad slab buffer through the k-quad tensor
 * map (csrc/tma.cuh), shared memory dumped to dst */
int fr_debug_tma_kquad(const float* src, float* dst, int WP, int ntiles, int tile, int g, fr_stream_t stream);

/* running count of kernels enqueued by this library (host-side counter) */
long long fr_kernel_launches(void);

const char* fr_last_error(void);
const char* fr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLOWREC_B200_H */
