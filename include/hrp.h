/*
 * hrp.h -- C ABI of libhrp, the B200-native hot path of arXiv 2405.08754
 * ("Hierarchical Resource Partitioning on Modern GPUs: A Reinforcement Learning Approach").
 *
 * Citations "P:<n>" are lines of the paper text; "R<n>" are the
 * readings of the paper listed in DESIGN.md.  The vocabulary follows Table I:
 * window W, concurrency limit Cmax, queue Q = {J_1..J_W}, job sets JS_i with partitionings
 * R_i, CoRunTime / SoloRunTime.
 *
 * Conventions (every entry point):
 *  - Returns hrp_status; HRP_OK = 0.  On error nothing is written to the outputs and
 *    hrp_last_error() returns a thread-local message.  Never aborts; no C++ exception crosses
 *    the ABI.
 *  - Pointers named d_* are caller-owned DEVICE pointers (e.g. torch tensor data_ptr) on the
 *    context's device; work is enqueued asynchronously on the context's CUDA stream (the one
 *    passed to hrp_env_create, NULL = legacy default stream).  Pointers without the prefix
 *    are HOST pointers, read synchronously and copied; the caller keeps ownership.
 *  - Input validation is synchronous (HRP_EINVAL / HRP_ERANGE).  CUDA / NCCL failures
 *    surface as HRP_ECUDA / HRP_ENCCL on the same or a later call, or from hrp_sync().
 *  - A context is not thread-safe.  Layout tables are generated on the host at create time.
 *  - Integer layouts: window pool ids are uint8 [n][W] row-major; scheduled-job sets are
 *    uint64 bitmasks (bit j = window position j); action indices are int64 (see
 *    hrp_decode_action for the index definition).
 */
#ifndef HRP_H
#define HRP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HRP_OK = 0,
  HRP_EINVAL = 1, /* null pointer / bad argument                                    */
  HRP_ENOMEM = 2, /* device or host allocation failed                               */
  HRP_ECUDA = 3,  /* CUDA runtime error (message has the CUDA error string)         */
  HRP_ENCCL = 4,  /* NCCL error                                                     */
  HRP_ERANGE = 5, /* size outside the supported range (W, Cmax, P, n, ...)          */
  HRP_ESTATE = 6, /* call not valid in the current state (e.g. replay < batch)      */
  HRP_ENUMERIC = 7 /* non-finite Q values met by a greedy argmax (from hrp_sync)     */
} hrp_status;

typedef struct hrp_ctx hrp_ctx; /* opaque: tables, weights, replay, workspaces, NCCL comm */

/* "Job Profiles Repository" as a pool table, indexed by pool id.  Host arrays,
 * copied at create.  Fields are the solo-run profile of each program: SoloRunTime on the
 * whole GPU and the Table III counters. */
typedef struct {
  int32_t n_jobs;            /* P, 1..256 (window entries are uint8 pool ids)            */
  int32_t n_features;        /* f, must be 12 (Table III lists 12 counters)              */
  const int64_t *solo_ticks; /* [P] solo run time T_p > 0, in ticks (1 tick = 1 us), <2^31 */
  const int16_t *compute_pm; /* [P] "Compute (SM) [%]" in permille, 1..1000               */
  const int16_t *memory_pm;  /* [P] "Memory [%]" in permille, 1..1000                     */
  const float *features;     /* [P][f] standardised counters (R11)                        */
} hrp_profiles;

/* One slot of a layout: a job's share of compute (1/800 GPU = GPCs x MPS percent) and of
 * memory bandwidth (1/8 GPU), and its memory domain (MIG GPU Instance). */
typedef struct {
  uint16_t sm800;
  uint8_t b8;
  uint8_t domain;
} hrp_slot;

/* The partition-configuration space R and the scheduling attributes W, Cmax
 * (Table I).  Layouts = MIG GI configs x maximal CI packings x MPS compositions with at most
 * Cmax slots, generated in the canonical order of DESIGN.md "Layout table" (R3-R6, R24). */
typedef struct {
  int32_t window;           /* W: 1..64                                                   */
  int32_t cmax;             /* Cmax: 1..4 and <= W                                        */
  uint32_t mps_split_mask;  /* bit k (1..19) set => MPS share 5k % allowed inside a CI    */
  int32_t mig;              /* 0: MIG-off (MPS-only) layouts; 1: also the 19 GI configs   */
  int32_t n_layouts;        /* 0: generate; >0: use the explicit table below (baselines)  */
  const int32_t *layout_nslots; /* [n_layouts] host, each 1..cmax                         */
  const hrp_slot *layout_slots; /* [n_layouts][4] host                                    */
  int32_t interference_q3;  /* co-runner memory interference in 1/8 units (R8; default 1)  */
} hrp_space;

typedef struct {
  int32_t n_envs;           /* E: environments on this rank, >= 1                          */
  int32_t batch;            /* B: replay batch on this rank, >= 1                          */
  int32_t replay_capacity;  /* N_rep >= max(batch, n_envs) (one step's E inserts must land  */
                            /* in distinct ring slots)                                     */
  int32_t hidden_layers;    /* d >= 1 (Table VI: fully connected + ReLU)                   */
  int32_t hidden_width;     /* w, multiple of 4, <= 1024                                   */
  float gamma;              /* discount                                            */
  float lr;                 /* SGD learning rate alpha                             */
  float reward_lambda;      /* r = r_f + lambda * sum r_i (Table VI, R9)                   */
  int32_t argmax_mode;      /* 0 auto (= 2), 1 explicit enumeration of every valid action  */
                            /* (W <= 16), 2 exact top-C pruned search; same actions bit    */
                            /* for bit (R15)                                    */
  /* SURVEY §8(f) row 4 variants (zero = the paper's defaults):                            */
  int32_t optimizer;        /* 0 plain SGD, 1 Adam (Kingma & Ba) with the three      */
  float adam_beta1, adam_beta2, adam_eps;   /* parameters below (bias-corrected moments)    */
  int32_t loss;             /* 0 (1/2) delta^2, 1 Huber with threshold huber_kappa:  */
  float huber_kappa;        /* h = delta^2/2 if |delta| <= kappa else kappa(|delta| - kappa/2) */
  int32_t precision;        /* 0 fp32-accurate 3xTF32 GEMMs; 1 fast mode: one TF32 MMA per   */
                            /* product (inputs rounded to tf32), policy-level parity only     */
  int32_t agent;            /* 0 joint agent (R1/R2: factorised duelling head over (l, g,     */
                            /* sigma)); 1 sequential agent (flat duelling */
                            /* head [v, a_l] with one advantage per partition setup, P:259's  */
                            /* "A = 29"; the job set is the next C_l jobs in queue order on   */
                            /* slots in order).  Actions keep the joint index.               */
} hrp_train_cfg;

/* ---- lifecycle ------------------------------------------------------------------------ */

/* Create a context on `device` with CUDA stream `cuda_stream` (cudaStream_t or NULL).
 * rank/world: this process's place among `world` data-parallel replicas (one per GPU);
 * nccl_unique_id: 128-byte ncclUniqueId from hrp_nccl_unique_id() on rank 0, broadcast by the
 * caller (required for world > 1; with world == 1 a non-NULL id builds a one-rank NCCL
 * communicator so that the allreduce path runs on one GPU -- a test configuration).  init_weights: host fp32 [hrp_n_params] online weights
 * (target := online), NULL = zeros.  Parameter layout: per Linear layer W [out][in]
 * row-major then b [out]; layer dims W*(f+5) -> w (x d) -> H = 1 + L + W*T (R1).
 * Errors: EINVAL, ERANGE (sizes), ENOMEM, ECUDA, ENCCL. */
hrp_status hrp_env_create(const hrp_space *space, const hrp_profiles *profiles,
                          const hrp_train_cfg *cfg, int device, void *cuda_stream, int rank,
                          int world, const void *nccl_unique_id, const float *init_weights,
                          hrp_ctx **out);
hrp_status hrp_env_destroy(hrp_ctx *ctx);
/* rank 0 helper: writes a 128-byte ncclUniqueId to `out` (host). */
hrp_status hrp_nccl_unique_id(void *out);

/* Load the first window of every env: d_windows uint8 [E][W]; all jobs unscheduled. */
hrp_status hrp_env_reset(hrp_ctx *ctx, const uint8_t *d_windows);

/* ---- the DQN step --------------------------------------- */

/* One vectorised environment step for all E envs:
 * encode the state, score every valid action with the online duelling Q-net,
 * take the argmax (ties -> lowest index, fixed-point Q^, R15), epsilon-greedy: explore iff
 * d_u_explore[e] < eps_threshold (thr = floor(eps * 2^32) in [0, 2^32]) and then take the
 * k-th valid action, k = floor(d_u_action[e] * n_valid / 2^64) (R14); compute
 * CoRunTime / SoloRunTime and r = (Solo/CoRun - 1)*100 + lambda*sum r_i (Table VI, P:258,
 * R7-R9); schedule the chosen jobs; write (s, a, r, done) to the replay ring at slot
 * (t*E + e) mod N_rep; envs whose jobs are all scheduled load d_next_windows[e] (R19).
 * Outputs (device): d_actions int64 [E], d_rewards f32 [E], d_done uint8 [E]; optional
 * (NULL = skip): d_corun int64 [E] CoRunTime ticks, d_qsel f32 [E] Q^(s, a) of the taken
 * action, d_greedy int64 [E] the greedy action (before epsilon). */
hrp_status hrp_env_step(hrp_ctx *ctx, uint64_t eps_threshold, const uint32_t *d_u_explore,
                        const uint64_t *d_u_action, const uint8_t *d_next_windows,
                        int64_t *d_actions, float *d_rewards, uint8_t *d_done,
                        int64_t *d_corun, float *d_qsel, int64_t *d_greedy);

/* Online inference (epsilon = 0): greedy action and its Q^ for n states given as
 * windows uint8 [n][W] + scheduled masks uint64 [n] (at least one job unscheduled).
 * d_argmax int64 [n], d_qmax f32 [n]; d_head f32 [n][H] optional raw head output z. */
hrp_status hrp_q_forward(hrp_ctx *ctx, int64_t n, const uint8_t *d_windows,
                         const uint64_t *d_sched, int64_t *d_argmax, float *d_qmax,
                         float *d_head);

/* One double-DQN update from B replay samples:
 * idx_b = floor(d_u_replay[b] * n_filled / 2^32); a* = argmax_online(s'); y = r +
 * gamma (1 - done) Q_target(s', a*); delta = Q_online(s, a) - y; L = sum delta^2 / (2B);
 * plain SGD on L with the gradient summed over all ranks / (B * world) (NCCL allreduce when
 * world > 1); if sync_target, target := online after the step.
 * d_loss f32 [1] (this rank's L); optional: d_sample_idx int64 [B], d_astar int64 [B]
 * (-1 where done).  Error ESTATE if fewer than B transitions were inserted. */
hrp_status hrp_dqn_update(hrp_ctx *ctx, const uint32_t *d_u_replay, int sync_target,
                          float *d_loss, int64_t *d_sample_idx, int64_t *d_astar);

/* Data-parallel building blocks of hrp_dqn_update:
 * hrp_dqn_grad runs the same update up to the backward and writes this rank's gradient of the
 * loss -- sum over its B samples of dL/dtheta, already scaled by 1 / (B * world) -- to d_grad
 * (device f32 [hrp_n_params], caller-owned) WITHOUT the NCCL allreduce and without changing the
 * weights; hrp_apply_grad then performs the SGD step theta -= lr * d_grad (+ target sync) with
 * any gradient, e.g. one summed over shards by the caller.  hrp_dqn_update == hrp_dqn_grad +
 * allreduce + hrp_apply_grad.  Same errors as hrp_dqn_update. */
hrp_status hrp_dqn_grad(hrp_ctx *ctx, const uint32_t *d_u_replay, float *d_loss,
                        int64_t *d_sample_idx, int64_t *d_astar, float *d_grad);
hrp_status hrp_apply_grad(hrp_ctx *ctx, const float *d_grad, int sync_target);

/* ---- exhaustive optimum ------------------------------ */

/* For each of n windows (uint8 [n][W], W <= 12): the minimum over set partitions of Q into
 * job sets of size <= Cmax of sum_i min_{R_i feasible} CoRunTime(JS_i, R_i), with
 * CoRun <= Solo per job set; canonical tie-break "block order" (R21b); each job
 * set's partitioning ties to the lowest action index.  Outputs (device): d_best_corun int64
 * [n] (the optimum), d_solo int64 [n] (time sharing), d_rgs uint8 [n][W] (job set of each
 * window position, sets numbered by their smallest position), d_block_action int64 [n][W]
 * (action index of each job set in set order, -1 padded).  Stateless and synchronous (returns
 * once the results are written); stream may be NULL. */
hrp_status hrp_bruteforce_optimum(const hrp_space *space, const hrp_profiles *profiles,
                                  int64_t n_windows, const uint8_t *d_windows,
                                  int64_t *d_best_corun, int64_t *d_solo, uint8_t *d_rgs,
                                  int64_t *d_block_action, void *cuda_stream);

/* The same search with the layout space's tables kept resident: hrp_brute_create validates
 * (the space must contain the whole-GPU single-slot layout, so that every window has a feasible
 * schedule: EINVAL otherwise)
 * and uploads them once (synchronous; errors as hrp_bruteforce_optimum), hrp_brute_run only
 * enqueues the search kernel on `cuda_stream` (asynchronous, no allocation, graph-capturable),
 * hrp_brute_destroy frees the tables (after the caller's work on them is complete).
 * hrp_bruteforce_optimum = create + run + synchronize + destroy. */
typedef struct hrp_brute hrp_brute;
hrp_status hrp_brute_create(const hrp_space *space, const hrp_profiles *profiles, int device,
                            void *cuda_stream, hrp_brute **out);
hrp_status hrp_brute_run(hrp_brute *plan, int64_t n_windows, const uint8_t *d_windows,
                         int64_t *d_best_corun, int64_t *d_solo, uint8_t *d_rgs,
                         int64_t *d_block_action, void *cuda_stream);
hrp_status hrp_brute_destroy(hrp_brute *plan);
/* Per-job co-run times (AppSlowdown; Fairness) of given actions on the
 * plan's space: for n (window uint8 [n][W], action int64 [n]) pairs, d_corun int64 [n] =
 * CoRunTime and d_solo int64 [n] = SoloRunTime of the action's job set (R7, R8), and
 * d_member_time int64 [n][4] = each member's own co-run time t_k -- member i is window position
 * g_i (ascending, hrp_decode_action's order), -1 padded; AppSlowdown = t_k / T_p.  An action
 * outside [0, |A|) gives -1 everywhere.  Asynchronous on cuda_stream. */
hrp_status hrp_job_times(hrp_brute *plan, int64_t n, const uint8_t *d_windows,
                         const int64_t *d_actions, int64_t *d_corun, int64_t *d_solo,
                         int64_t *d_member_time, void *cuda_stream);

/* ---- host helpers (no device work) ---------------------------------------------------- */

/* Layout table of `space` (host): n_layouts, per layout its slot count and slots in slot
 * order, per slot its type id (types = distinct (sm800, b8), ascending), n_types, and the
 * action count |A| = sum_l P(W, C_l) (P:315 + the C = 1 term).  Arrays have room for `cap`
 * layouts; ERANGE if more are needed (n_layouts is still written). */
hrp_status hrp_layout_table(const hrp_space *space, int32_t cap, int32_t *n_layouts,
                            int32_t *layout_nslots, hrp_slot *slots /*[cap][4]*/,
                            uint8_t *slot_type /*[cap][4]*/, int32_t *n_types,
                            int64_t *n_actions);

/* Decode action index idx = off[l] + rank_lex(g) * C! + lehmer(sigma) into the layout l,
 * the window positions g[0] < ... < g[C-1] and slot_of[i] = sigma(i) (member i -> slot);
 * unused entries are -1.  ERANGE if idx is outside [0, |A|). */
hrp_status hrp_decode_action(const hrp_space *space, int64_t idx, int32_t *l, int32_t g[4],
                             int32_t slot_of[4]);

int64_t hrp_n_params(const hrp_ctx *ctx);  /* parameters of ONE network, -1 if ctx NULL */
/* Test hook: rows [0, rows) of hidden layer `layer`'s output (0-based, ReLU applied) from the
 * most recent online forward, as the backward's ReLU' mask reads them (tf32 hi plane: same sign
 * as the fp32 value) -> d_out f32 [rows][w] (device).  After hrp_dqn_update / hrp_dqn_grad the
 * rows [0, B) are the sampled states s.  Used by the parity tests for reading R25. */
hrp_status hrp_get_hidden(hrp_ctx *ctx, int layer, int64_t rows, float *d_out);
int32_t hrp_head_width(const hrp_ctx *ctx); /* H */
/* Host copies of the flat fp32 weights: out [2 * n_params] = online | target. */
hrp_status hrp_get_weights(hrp_ctx *ctx, float *out);
hrp_status hrp_set_weights(hrp_ctx *ctx, const float *in /*[2 * n_params]*/);
/* Number of libhrp kernel launches enqueued so far by this context (for bench.py). */
int64_t hrp_launch_count(const hrp_ctx *ctx);
/* Per-kernel device timing: with profiling enabled every libhrp launch on the context's
 * stream is bracketed by CUDA events; hrp_profile_read synchronises and returns the summed
 * milliseconds and launch counts per kernel class (arrays of HRP_K_COUNT, host). */
typedef enum {
  HRP_K_ENCODE = 0,   /* a2 state encoding                                          */
  HRP_K_GEMM_FWD = 1, /* a3 Q-MLP forward GEMMs (+ fused bias / ReLU)                */
  HRP_K_GEMM_BWD = 2, /* a11 backward GEMMs, split-K reduce, bias column sums         */
  HRP_K_SELECT = 3,   /* a4-a7 fused centering / argmax / epsilon / reward / replay   */
  HRP_K_TD = 4,       /* a9-a10 double-DQN target argmax, TD error, head gradient     */
  HRP_K_SAMPLE = 5,   /* a8 replay sample                                            */
  HRP_K_SGD = 6,      /* a13 SGD + target sync                                        */
  HRP_K_MISC = 7,     /* loss reduction                                             */
  HRP_K_ALLREDUCE = 8,/* a12 NCCL gradient allreduce (world > 1)                      */
  HRP_K_HEAD_BWD = 9, /* a10-a11 structured duelling-head backward (gathers / scatters) */
  HRP_K_COUNT = 10
} hrp_kernel_class;
hrp_status hrp_profile(hrp_ctx *ctx, int enable); /* 1: clear + start recording; 0: stop */
hrp_status hrp_profile_read(hrp_ctx *ctx, double *ms, int64_t *launches);
/* Explicit Q^ evaluations (valid (l, g, sigma) scored; pruned mode: candidate assignments)
 * counted by the selection kernels since create (synchronises the stream). */
int64_t hrp_eval_count(hrp_ctx *ctx);
/* The same count split by kernel: out[0] = env step / inference selection, out[1] = the
 * double-DQN target argmax of hrp_dqn_update (host int64 [2]; synchronises the stream). */
hrp_status hrp_eval_counts(hrp_ctx *ctx, int64_t *out);
/* Valid actions covered by the exact argmax since create -- every valid (l, g, sigma) of each
 * state whose greedy action was computed (the explicit enumeration's evaluations; the pruned
 * search reaches the same maximum without scoring them one by one): out[0] env step /
 * inference, out[1] the double-DQN target argmax (host int64 [2]; synchronises the stream). */
hrp_status hrp_covered_counts(hrp_ctx *ctx, int64_t *out);
/* Diagnostics: one tensor-core GEMM D[M][N] = A[M][K] . W[N][K]^T + bias (3xTF32, the Q-MLP
 * forward kernel) on `device` / `cuda_stream`, all pointers device; d_trace (optional,
 * uint64 [256]) receives %globaltimer stamps of CTA (0,0): [0] start, [1] setup, [2+kb] TMA
 * issue, [130+kb] MMA issued, [194] accumulator ready, [195] end.  With reps > 0 and ms_out,
 * *ms_out = the average device time of `reps` further back-to-back GEMM launches (operands
 * already split).  force_bn: output tile width 64 / 128 / 256, 0 = the library's choice. */
hrp_status hrp_diag_gemm(int device, void *cuda_stream, int M, int N, int K, const float *d_A,
                         const float *d_W, const float *d_bias, float *d_D,
                         uint64_t *d_trace, int reps, int force_bn, float *ms_out);
/* Diagnostics: ALU issue-rate microbenchmark on `device` -- 148 x 8 CTAs of 256 threads, each
 * thread 8 independent chains of `iters` x 16 fp32 adds (is_int = 0) or int32 adds (1);
 * *lane_ops_per_s = adds / second (the roofline peak of the selection kernels). */
hrp_status hrp_diag_alu(int device, int is_int, int iters, double *lane_ops_per_s);
/* Diagnostics (process-wide, for A/B measurements): key 0 = TMEM accumulator layout of the
 * tensor-core GEMMs: 0 one accumulator for all three 3xTF32 products, 1 the hi.hi products in
 * one accumulator and the hi.lo + lo.hi corrections in another, 2 (default) the hi.hi products
 * spread round-robin by K block over up to three accumulators plus the correction one. */
hrp_status hrp_diag_config(int key, int value);
/* Block until the context's stream is idle; returns any pending CUDA/NCCL error, or
 * HRP_ENUMERIC (once, then cleared) if a greedy argmax since the last call met non-finite Q
 * values (e.g. diverged weights); such a state took its lowest valid action instead. */
hrp_status hrp_sync(hrp_ctx *ctx);
const char *hrp_last_error(void);
const char *hrp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HRP_H */
