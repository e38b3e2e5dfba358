/*
 * pod.h — C ABI of libpod.so, the B200-native (sm_100a) hot path of
 * FinRL-Podracer (arXiv 2111.05188): a massively vectorised stock-trading
 * rollout, its GAE scan and generational-evolution elite selection.
 *
 * Citations: "P:Lx" = PAPER.md line x (/root/reference, LaTeX source of the
 * paper); "S:Lx" = SPEC.md line x; "R#k" = reading k in DESIGN.md §3.
 *
 * Conventions for every entry point
 *   - Plain C types only.  Pointers marked [dev] are CUDA device pointers, [host]
 *     are host pointers.  `stream` is a cudaStream_t passed as void*.
 *   - The CALLER owns all device memory (market tensors, workspace,
 *     trajectories, actor parameters, outputs).  The library owns only the
 *     opaque handles, the TMA descriptors and CUDA graphs cached in them, and
 *     the NCCL communicator.  Nothing is allocated inside a hot call
 *     (pod_rollout, pod_gae, pod_select_elite).
 *   - Calls are stream-ordered and asynchronous unless stated otherwise; a
 *     buffer must stay alive until the stream work that uses it completes.
 *   - Every function returns a pod_status.  Argument errors are detected on
 *     the host and returned synchronously without launching anything; the
 *     thread-local pod_last_error() gives a one-line reason.  Device-side
 *     faults (non-finite actor mean or account value) set a device error word
 *     that pod_env_check() and pod_env_read_state() turn into
 *     POD_ERR_NONFINITE.
 *   - A handle is not thread-safe; distinct handles are independent.
 *   - Compute capability must be 10.0 (B200, sm_100a): there is no fallback
 *     path of any kind (POD_ERR_UNSUPPORTED otherwise).
 */
#ifndef POD_H
#define POD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POD_ABI_VERSION 3
#define POD_ENV_TILE 32      /* envs per tile: one warp; a tile shares its episode start row */
#define POD_MAX_HIDDEN_LAYERS 4

typedef enum {
    POD_OK = 0,
    POD_ERR_ARG = 1,          /* bad scalar argument or NULL where required            */
    POD_ERR_SHAPE = 2,        /* inconsistent or unsupported sizes                      */
    POD_ERR_RANGE = 3,        /* start row out of range of the market data */
    POD_ERR_WORKSPACE = 4,    /* workspace too small or misaligned                      */
    POD_ERR_CUDA = 5,         /* a CUDA runtime/driver call failed                      */
    POD_ERR_NCCL = 6,         /* NCCL missing or a collective failed                    */
    POD_ERR_NONFINITE = 7,    /* non-finite mean action / account value / fitness       */
    POD_ERR_UNSUPPORTED = 8   /* device is not sm_100, or a shape outside kernel limits */
} pod_status;

const char* pod_status_string(pod_status s);
/* Detail of the last failing call on this thread ("" if none). */
const char* pod_last_error(void);
int pod_abi_version(void);
/* Measurement support: the number of kernels this library has launched in this
 * process (every entry point; a launch of a cached CUDA graph counts the graph's
 * kernel nodes), e.g. sampled around a timed region. */
unsigned long long pod_kernel_launches(void);

typedef struct pod_env pod_env_t;    /* opaque */
typedef struct pod_comm pod_comm_t;  /* opaque */

/* Environment configuration (§3; defaults).
 *   n_envs          N, envs on this process/GPU (>= 1; ragged last tile allowed)
 *   n_stocks        n (1..102 with n_feat = 3: obs_dim = 1+2n+nf must be <= 512)
 *   n_feat          f indicator channels (3 = MACD, RSI, CCI)
 *   n_agents        P_local; envs are split into n_agents contiguous equal groups,
 *                   group a acts with agent a's parameters (N % n_agents == 0)
 *   horizon         H, episode length in steps (R#10)
 *   h_max           max shares per ticker per step (R#7; >= 1)
 *   env_offset      global id of env 0 — the Philox counter uses global env ids so
 *                   results do not depend on the GPU count (R#14)
 *   initial_capital C0 > 0 (P:L415 $1,000,000)
 *   cost_rate       c in [0,1) of traded notional, both sides (P:L415 0.2%, R#1–2)
 *   reward_scale    r = reward_scale * (v_{t+1} - v_t) (R#8)
 *   gamma           discount in (0,1] for the fitness J (Eq. 1)
 *   seed            Philox key for the action noise (R#14)                         */
typedef struct {
    int32_t n_envs;
    int32_t n_stocks;
    int32_t n_feat;
    int32_t n_agents;
    int32_t horizon;
    int32_t h_max;
    int64_t env_offset;
    double initial_capital;
    double cost_rate;
    double reward_scale;
    double gamma;
    uint64_t seed;
} pod_env_config;

/* Market tensors [dev], float32, row-major, immutable while a handle uses them:
 *   close [T_data][n] > 0 closing prices p_t
 *   feat  [T_data][f][n] indicator channels, channel-major, pre-scaled (R#9)   */
typedef struct {
    const float* close;
    const float* feat;
    int64_t T_data;   /* 2 <= T_data < 2^31 */
} pod_market;

/* Actor MLP parameters [dev] ("policy ... maps a state to an action
 * vector over n stocks"; Gaussian head R#12; hidden activation R#13).
 * `params` holds n_agents contiguous slabs of param_bytes each, laid out as
 * pod_actor_layout() reports: bf16 weight matrices W_l[out][in_pad] (row-major,
 * K-major for the tensor cores; pad columns/rows must be finite, zero is
 * recommended), then float32 biases and float32 log_std.  param_bytes must be
 * >= layout.param_bytes and a multiple of 16; params must be 16-byte aligned. */
typedef struct {
    int32_t n_hidden;   /* 1..POD_MAX_HIDDEN_LAYERS */
    int32_t hidden;     /* 64, 128, 192, 256 or 512 */
    int32_t act;        /* 0 = ReLU, 1 = tanh       */
    int32_t reserved;
    const void* params;
    size_t param_bytes;
} pod_actor;

typedef struct {
    int32_t obs_dim;       /* 1 + 2n + n f                                   */
    int32_t k_pad;         /* obs_dim rounded up to 64 (obs row stride)       */
    int32_t n_out_pad;     /* n + 1 rounded up to 32 (head rows: 0..n-1 the  *
                            * action means, row n the critic V, R#22)         */
    int32_t n_layers;      /* n_hidden + 1                                    */
    size_t w_offset[POD_MAX_HIDDEN_LAYERS + 1];   /* bytes, bf16 [out_l][in_l] */
    int32_t w_rows[POD_MAX_HIDDEN_LAYERS + 1];    /* out_l (padded)            */
    int32_t w_cols[POD_MAX_HIDDEN_LAYERS + 1];    /* in_l  (padded)            */
    size_t b_offset[POD_MAX_HIDDEN_LAYERS + 1];   /* bytes, float32 [out_l]    */
    size_t log_std_offset;                        /* bytes, float32 [n_out_pad] */
    size_t param_bytes;                           /* minimal slab size, %1024==0 */
    size_t n_elems;        /* parameters per slab incl. padding: sum rows*cols + sum rows + n_out_pad
                            * (the float32 vector pod_fuse_pods works on, same order as the slab) */
} pod_actor_layout;

/* Trajectory buffers [dev] (transitions stay as tensors in
 * contiguous GPU memory).  T = rollout length, N = n_envs.
 *   obs      bf16 [T+1][N][k_pad]  s_0..s_T; pad columns written as 0     (required)
 *   act      f32  [T][N][n]        raw (pre-tanh) sampled action          (required unless injected)
 *   logp     f32  [T][N]           log pi(raw | s_t)                      (required unless injected)
 *   rew      f32  [T][N]           r_t (Eq. 2, R#8)                       (required)
 *   done     u8   [T][N]           episode ended at this transition       (required)
 *   mu       f32  [T][N][n]        actor mean                             (optional, NULL)
 *   dbg_aint i16  [T][N][n]        executed integer action a_t            (optional)
 *   dbg_hold i32  [T][N][n]        h_{t+1} after the trade, before reset  (optional)
 *   dbg_cash f64  [T][N]           b_{t+1} after the trade, before reset  (optional)
 *   equity   f64  [T][N]           account value v_{t+1} = b + p_{t+1}^T h after
 *                                  step t, before any auto-reset (the backtest
 *                                  curve, R#25)                            (optional)
 *   val      f32  [T+1][N]         critic V(s_t), t = 0..T: head row n over the
 *                                  actor's trunk (R#22); val[T] = V(s_T), the
 *                                  GAE bootstrap, from one extra value-only
 *                                  actor pass.  Feeds pod_gae directly.  (optional) */
typedef struct {
    uint16_t* obs;
    float* act;
    float* logp;
    float* rew;
    uint8_t* done;
    float* mu;
    int16_t* dbg_aint;
    int32_t* dbg_hold;
    double* dbg_cash;
    float* val;
    double* equity;
} pod_traj;

/* ---------------------------------------------------------------- layout */
/* Parameter-slab layout for an actor over this config's observation (host
 * only, no device work).  Errors: POD_ERR_ARG / POD_ERR_UNSUPPORTED. */
pod_status pod_actor_layout_get(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                                pod_actor_layout* out);

/* ----------------------------------------------------------- environment */
/* Bytes of device workspace a handle for `cfg` needs (host only). */
pod_status pod_env_workspace_size(const pod_env_config* cfg, size_t* bytes);

/* Validate cfg (S:L139 invariants: C0 > 0, 0 <= c < 1, h_max >= 1,
 * 0 < gamma <= 1), check the device is sm_100, and bind market + workspace
 * (ws [dev], >= pod_env_workspace_size bytes, 256-byte aligned).  The market
 * is scanned once on the device (synchronously): every close price must be
 * finite and > 0 and every indicator finite, else POD_ERR_NONFINITE.  The env
 * state is undefined until pod_env_reset.  Errors: ARG, SHAPE, WORKSPACE,
 * UNSUPPORTED, NONFINITE, CUDA. */
pod_status pod_env_create(const pod_env_config* cfg, const pod_market* market, void* ws,
                          size_t ws_bytes, pod_env_t** out);
pod_status pod_env_destroy(pod_env_t* env);

/* Reset every env (R#17): b = C0, h = 0, k = 0, t = s, where s is
 * the episode start row of the env's tile.
 *   tile_start_rows [host] int64 [ceil(N/32)], each with s + H <= T_data - 1
 *                   (else POD_ERR_RANGE); NULL = draw them from the config seed.
 *   obs0            [dev] bf16 [N][k_pad] or NULL: also write s_0.
 * Resets the action-noise step counter to 0.  Stream-ordered. */
pod_status pod_env_reset(pod_env_t* env, const int64_t* tile_start_rows, uint16_t* obs0, void* stream);

/* Run T >= 1 lockstep steps of all envs (a batched environment that
 * takes a batch of actions and returns a batch of transitions).  Per step t:
 *   1. actor mean mu = MLP(s_t) on tcgen05 tensor cores (bf16 x bf16 -> f32),
 *      raw = mu + exp(log_std) z, z ~ N(0,1) from Philox4x32-10 +
 *      Box–Muller (R#12, R#14), logp, u = tanh(raw), a = sgn(u) floor(|u| h_max
 *      + 1/2) (R#6);  deterministic != 0: raw = mu (z = 0);
 *      injected_u [dev] f32 [T][N][n] in [-1,1] (or NULL) replaces 1. by a = map(u)
 *      and leaves act/logp/mu untouched;
 *   2. env step (Eqs. 3–4, reward Eq. 2, readings R#1–5, R#18):
 *      sells then greedy buys in ticker order with a float64 cash ledger,
 *      r = scale (v' - v), done = (k+1 == H) or (t+1 == T_data-1), auto-reset
 *      with the terminal transition reported;
 *   3. s_{t+1} written to obs[t+1].
 * With traj.val (sampled or deterministic mode), step t also writes the critic
 * value V(s_t) from the same MLP pass (head row n), and one value-only actor
 * pass over obs[T] writes val[T].
 * obs[0] is first written from the carried state, so buffers need not persist
 * across calls; obs[T] is the bootstrap state.  fitness_out [dev] f64
 * [n_agents] or NULL: afterwards J_a = mean over agent a's envs of the
 * discounted return of each env's last completed episode (Eq. 1, R#15).
 * Execution (results identical either way): when every 128-env M-tile's CTA
 * pair fits on the device at once (2 x M-tiles <= SMs), agents hold whole
 * M-tiles (N / n_agents % 128 == 0), one env group, no injected actions and
 * no profiling, the T steps run as ONE launch in which each CTA pair runs the
 * actor and the env step of its 128 envs for all steps (the rollout_fused
 * kernel; POD_FUSED=0 in the environment at pod_env_create turns it off);
 * otherwise as 2T launches (actor, env step).  Each rollout first copies the
 * actor's weights into ring-stage order in a device buffer the handle
 * allocates on first use (n_agents x the weight bytes of the slab; freed by
 * pod_env_destroy; POD_WT=0 at pod_env_create streams from the slab instead).
 * Errors (host, synchronous): ARG, SHAPE, UNSUPPORTED, CUDA. */
pod_status pod_rollout(pod_env_t* env, const pod_actor* actor, int32_t T, const pod_traj* traj,
                       const float* injected_u, int32_t deterministic, double* fitness_out,
                       void* stream);

/* Per-kernel device timing (measurement support, not part of the method).
 * stride k > 0: subsequent pod_rollout calls run the separate actor / env-step
 * launches (not the fused rollout kernel) and record CUDA events around the
 * actor launches and the env-step launches of every k-th step, on the stream
 * (graph branch) each launch runs on; 0 turns it off.  pod_env_profile_read
 * synchronises `stream` and returns, for the most recent profiled rollout, the
 * summed device milliseconds of the bracketed launches and their size in
 * "units" (sum over bracketed launches of envs-in-launch / n_envs; a launch
 * over all envs counts 1), then forgets it (zeros if none since the last read).
 * Note: with env groups (pod_rollout runs 2 independent halves of the envs on
 * separate graph branches so one half's env step overlaps the other's actor)
 * the bracketed launches may overlap in time. */
pod_status pod_env_profile(pod_env_t* env, int32_t stride);
pod_status pod_env_profile_read(pod_env_t* env, double* actor_ms, double* actor_units, double* env_ms,
                                double* env_units, void* stream);

/* Diagnostics only: actor_buf [dev] u64 [2 x M-tiles][64] receives clock64 stamps of
 * the actor kernel's phases (obs loaded, per-layer MMA issue / epilogue, head) and
 * env_buf [dev] u64 [env tiles][8] those of the env-step kernel (start, inputs staged,
 * sells done, buys done, ledger done, rows staged, end) at every launch of
 * subsequent rollouts; NULL turns either off.  Drops cached graphs. */
pod_status pod_debug_trace(pod_env_t* env, unsigned long long* actor_buf, unsigned long long* env_buf);

/* Fitness J of the current state (same definition as pod_rollout's). */
pod_status pod_env_fitness(pod_env_t* env, double* fitness_out, void* stream);

/* Copy the carried state to caller buffers [dev] (any may be NULL):
 * hold i32 [N][n] (env-major), cash/asset/ep_ret f64 [N].  Synchronises the
 * stream and returns POD_ERR_NONFINITE if the device error word is set. */
pod_status pod_env_read_state(pod_env_t* env, int32_t* hold, double* cash, double* asset,
                              double* ep_ret, void* stream);

/* Synchronise `stream` and report (then clear) the device error word. */
pod_status pod_env_check(pod_env_t* env, void* stream);

/* ---------------------------------------------------------------- GAE */
/* Generalised advantage estimation over [T][N] (R#11; PPO P:L472):
 *   delta_t = r_t + gamma (1-d_t) V_{t+1} - V_t,  V_T = boot,
 *   A_t = delta_t + gamma lambda (1-d_t) A_{t+1}, A_T = 0,  R_t = A_t + V_t.
 * rew, val f32 [T][N], done u8 [T][N], boot f32 [N] -> adv, ret f32 [T][N], all
 * [dev], row-major (time-major).  T, N >= 1.
 * adv_stats [dev] f64 [2] or NULL: per-buffer advantage normalisation (S:L278,
 * R#23): the scan also accumulates S1 = sum A, S2 = sum A^2 (float64) into
 * adv_stats (zeroed first), then adv is rewritten in place as (A - m) / s with
 * m = S1/(T N), s = sqrt(S2/(T N) - m^2) (all zeros if s == 0); ret keeps the
 * unnormalised A_t + V_t.  Stream-ordered, no host synchronisation.
 * Errors: ARG, CUDA. */
pod_status pod_gae(const float* rew, const float* val, const uint8_t* done, const float* boot,
                   int32_t T, int32_t N, float gamma, float lambda, float* adv, float* ret,
                   double* adv_stats, void* stream);

/* ------------------------------------------------------ K-pod ensemble fusion */
/* Fuse the K pods of each agent once per epoch ("fusing the trained
 * models from K pods at each epoch"; P:L372 parameters, not gradients, are
 * exchanged, using the soft update; R#24):
 *   mean = (1/K) sum_pods theta,  fused = tau mean + (1 - tau) prev,
 *   every pod's theta <- fused, prev <- fused.
 * The pods of agent a are its K_local consecutive slots a*K_local .. +K_local-1
 * of `params` on every rank of `comm` (comm NULL: this process only), so
 * K = K_local * nranks.  params [dev] [P_local][param_bytes] slabs in the
 * pod_actor_layout of (cfg, n_hidden, hidden), in/out; bf16 weights are
 * rounded to nearest even from the float32 result.  prev [dev] f32
 * [P_local/K_local][layout.n_elems] the previous fused parameters (in/out);
 * may be NULL only when tau == 1 (hard adoption, S:L368 default).  work: not
 * used (kept for ABI compatibility; may be NULL).  tau in [0, 1].
 * One kernel per rank: the local pod sum (float32, pod order) is published in
 * a buffer every rank maps (CUDA IPC over NVLink, set up collectively on the
 * first call and whenever a larger one is needed), every rank waits for the
 * others' partials chunk by chunk, sums them in rank order (so every rank holds
 * bit-identical fused parameters), blends and narrows into its pods; no
 * collective library call.  Collective over `comm` (same arguments on every
 * rank), stream-ordered.  Errors: ARG, SHAPE, UNSUPPORTED, NCCL (setup), CUDA. */
pod_status pod_fuse_pods(pod_comm_t* comm, const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                         void* params, size_t param_bytes, int32_t P_local, int32_t K_local, float tau,
                         float* prev, float* work, void* stream);

/* Workspace bytes of pod_fuse_pods_local_ranks for R ranks (host only). */
pod_status pod_fuse_workspace_size(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden, int32_t P_local,
                                   int32_t K_local, int32_t R, size_t* bytes);

/* The same fusion over R (1..16) ranks' slab arrays that all live on this
 * device, in one launch whose block rows play the ranks and exchange their
 * partial sums through `ws` exactly as pod_fuse_pods' ranks do through peer
 * memory (the single-process multi-learner form, and the one-device check of
 * the cross-rank protocol).  params [host] R device pointers, each
 * [P_local][param_bytes]; prev [host] R device pointers (f32
 * [P_local/K_local][n_elems]) or NULL when tau == 1; K = K_local * R.
 * ws [dev] >= pod_fuse_workspace_size bytes, 256-byte aligned.
 * Stream-ordered.  Errors: ARG, SHAPE, WORKSPACE, UNSUPPORTED, CUDA. */
pod_status pod_fuse_pods_local_ranks(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden, void* const* params,
                                     size_t param_bytes, int32_t R, int32_t P_local, int32_t K_local, float tau,
                                     float* const* prev, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ PPO update */
/* Learner hyper-parameters (P:L472 PPO; Table 3 via S:L239–241; R#26). */
typedef struct {
    float ratio_clip;      /* epsilon, Table 3 "Ratio clip (PPO)" 0.25        */
    float entropy_coef;    /* Table 3 "Lambda entropy (PPO)" 0.02            */
    float value_coef;      /* 0.5 (S:L239 design decision)                   */
    float learning_rate;   /* Table 3 2^-14                                  */
    float adam_beta1;      /* 0.9                                            */
    float adam_beta2;      /* 0.999                                          */
    float adam_eps;        /* 1e-8                                           */
    int32_t fp32_operands; /* 0: bf16 operands on the tcgen05 tensor cores (the
                            * rollout slab's weights, bf16 activations / deltas,
                            * f32 accumulate); 1: float32 operands on the float32
                            * reference core (master weights; for parity checks) */
} pod_ppo_hparams;

/* Workspace bytes of pod_ppo_update for minibatches of `batch` rows (host). */
pod_status pod_ppo_workspace_size(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden, int32_t batch,
                                  size_t* bytes);

/* PPO clipped-surrogate update of one agent (R#26), on
 * the device buffers of a rollout: for each of the n_minibatches minibatches
 * (rows perm[j*batch .. (j+1)*batch) of the flattened buffer; the caller
 * shuffles and concatenates repeat_times permutations), with
 *   rho = exp(logp_theta(raw | s) - logp_old),
 *   L = -mean[min(rho A, clip(rho, 1-eps, 1+eps) A)] - c_ent H(pi)
 *       + c_v mean[(V(s) - R)^2],   H(pi) = sum_i (log sigma_i + (1 + ln 2 pi)/2),
 * the gradient of L (forward + backward as this library's GEMM kernels: with
 * hp->fp32_operands == 0, bf16 x bf16 -> float32 on the tcgen05 tensor cores,
 * the weights being the bf16 rollout slab, kept equal to the rounded float32
 * master after every step; with 1, float32 operands on the CUDA cores) and one
 * Adam step (bias-corrected, step t = adam_t + j + 1):
 *   m <- b1 m + (1-b1) g,  v <- b2 v + (1-b2) g^2,
 *   theta <- theta - lr (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps).
 * A minibatch whose loss is not finite (divergence) sets the
 * workspace's error word and is not applied (nor are the call's later
 * minibatches); pod_ppo_check reports it, and the next pod_ppo_update on the
 * same workspace returns POD_ERR_NONFINITE until pod_ppo_check has cleared it.
 * Afterwards the agent's rollout slab `params` (pod_actor_layout; agent 0 of
 * the slab array) is rewritten from theta (bf16 weights, RNE).
 *   master, adam_m, adam_v [dev] f32 [layout.n_elems] (pod_fuse_pods order), in/out;
 *   obs [dev] bf16 [M][k_pad], act_raw f32 [M][n], logp_old, adv, ret f32 [M]
 *   (traj.obs rows 0..T-1, traj.act, traj.logp, normalised advantages, returns);
 *   perm [dev] i32 [n_minibatches * batch] row indices in [0, M) (may be NULL
 *   when n_minibatches == 0: the call then only re-narrows master into params);
 *   losses [dev] f64 [4] accumulates (sum of the surrogate objective, sum of
 *   (V - R)^2, entropy per minibatch, rows); grad_out [dev] f32 [n_elems] or
 *   NULL: the last minibatch's gradient (diagnostics); ws >=
 *   pod_ppo_workspace_size (the last 256 bytes hold the device Adam step base).
 * The minibatch loop is captured into a CUDA graph on the first call with a
 * given set of pointers and sizes (adam_t, the hyper-parameters and the stream
 * excepted: they are passed through device memory, so schedules replay the same
 * graph) and replayed by later calls (library-owned, 16 per thread,
 * least recently used evicted); the first call on a workspace allocates its
 * 4-byte pinned error mirror.  All scratch lives in `ws`, so learners with
 * distinct buffers may run concurrently on different streams.
 * POD_PPO_GRAPH=0 launches eagerly instead.  Stream-ordered.
 * Errors: ARG, SHAPE, UNSUPPORTED, CUDA, NONFINITE (an earlier loss, above). */
pod_status pod_ppo_update(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden, int32_t act,
                          const pod_ppo_hparams* hp, float* master, float* adam_m, float* adam_v, int64_t adam_t,
                          void* params, size_t param_bytes, const uint16_t* obs, const float* act_raw,
                          const float* logp_old, const float* adv, const float* ret, int64_t M,
                          const int32_t* perm, int32_t batch, int32_t n_minibatches, double* losses,
                          float* grad_out, void* ws, size_t ws_bytes, void* stream);

/* Synchronise `stream`, then report (and clear) the learner error word of
 * workspace `ws`: POD_ERR_NONFINITE if a minibatch loss of an earlier
 * pod_ppo_update on it was not finite (the caller aborts the pod). */
pod_status pod_ppo_check(void* ws, void* stream);

/* ----------------------------------------------------------- evaluator */
/* Backtest metrics of one account-value curve per env (§5.2
 * "cumulative return ... annual return ... annual volatility ... Sharpe ratio
 * ... max drawdown"; R#25): v_0 = v0[e], v_t = curve[t-1][e] for
 * t = 1..T (one episode: a deterministic rollout whose horizon covers T, e.g.
 * traj.equity), rho_t = v_t / v_{t-1} - 1:
 *   out[0][e] cumulative return (v_T - v_0) / v_0
 *   out[1][e] annual return (v_T / v_0)^(ppy / T) - 1
 *   out[2][e] annual volatility std(rho) sqrt(ppy)   (sample, n - 1; 0 if T < 2)
 *   out[3][e] Sharpe (mean(rho) - rf) / std(rho) sqrt(ppy); NaN if std = 0 or T < 2
 *   out[4][e] max drawdown min_t (v_t / max_{s<=t} v_s - 1)   (<= 0)
 * v0 [dev] f64 [N], curve [dev] f64 [T][N], out [dev] f64 [5][N]; float64
 * throughout.  T >= 1, ppy > 0.  Errors: ARG, CUDA. */
pod_status pod_backtest_metrics(const double* v0, const double* curve, int32_t T, int32_t N,
                                double periods_per_year, double rf_per_period, double* out, void* stream);

/* Early-stop rule of the evaluator ("stop the training process using
 * the early stopping mechanism", "keeps track of the best agent so far";
 * S:L441–448; R#25), host only: best = argmax of history (earliest wins);
 * stop = 1 when the latest entry is at least `patience` entries after best.
 * Errors: ARG (empty history, patience < 0, NULL). */
pod_status pod_early_stop(const double* history, int32_t len, int32_t patience, int32_t* stop, int32_t* best);

/* -------------------------------------------------- generational evolution */
/* Selector plan ("redistributes the agents with the highest scores to
 * form a new population", R#16), host only: rank agents by
 * (J desc, id asc); the first k are elites and keep their parameters; the
 * eliminated slots, in ascending id, take elites in rank order, round-robin.
 * fitness [host] f64 [P_total] -> plan [host] i32 [P_total] (source agent
 * of every slot).  Errors: ARG (k outside [1,P_total], P_total < 1),
 * NONFINITE. */
pod_status pod_elite_plan(const double* fitness, int32_t P_total, int32_t k, int32_t* plan);

/* One parameter-slab transfer of a plan, as seen from `rank`:
 * kind 0 = local device copy src_local -> dst_local (before the exchange),
 * 1 = send slab src_local to `peer`, 2 = receive into dst_local from `peer`,
 * 3 = local device copy src_local -> dst_local after the exchange (fan-out of
 * a slab this rank received from `peer`).  Global agent g lives on rank
 * g / P_local at local index g % P_local.  An elite slab crosses to another
 * rank at most once per destination rank (k = 1: one copy per rank, a
 * broadcast), however many of that rank's slots take it. */
typedef struct {
    int32_t kind;
    int32_t peer;
    int32_t src_local;
    int32_t dst_local;
} pod_transfer;

/* Transfers `rank` must execute to realise `plan` (host only), in execution
 * order: kinds 0, then the sends/receives (one NCCL group), then kind 3.  Sends
 * and receives between a pair of ranks appear in the same (ascending slot)
 * order on both sides.  *n_ops gets the count; POD_ERR_ARG if max_ops is too
 * small or the plan is not a valid elite plan. */
pod_status pod_elite_transfers(const int32_t* plan, int32_t P_total, int32_t P_local, int32_t rank,
                               pod_transfer* ops, int32_t max_ops, int32_t* n_ops);

/* NCCL communicator over one process per GPU (libnccl.so.2 is loaded at
 * pod_comm_init; the torch process group only carries the 128-byte id). */
pod_status pod_comm_unique_id(uint8_t id[128]);
pod_status pod_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank,
                         int32_t max_agents_local, pod_comm_t** out);
pod_status pod_comm_destroy(pod_comm_t* comm);

/* One generation's selection step across all ranks:
 *   1. ncclAllGather of fitness_local [dev] f64 [P_local] -> [P_total];
 *   2. one stream synchronisation and a D2H copy of P_total doubles;
 *   3. the identical pod_elite_plan on every rank, written to h_plan [host]
 *      i32 [P_total];
 *   4. grouped ncclSend/ncclRecv (+ local cudaMemcpyAsync) moving elite
 *      parameter slabs into the eliminated slots of params [dev]
 *      [P_local][param_bytes] ("sending the network parameters"):
 *      one transfer per (elite, destination rank), then local fan-out copies
 *      (pod_elite_transfers).
 * Synchronous w.r.t. the plan (step 2), asynchronous for the slab moves.
 * Errors: ARG, NONFINITE, NCCL, CUDA. */
pod_status pod_select_elite(pod_comm_t* comm, const double* fitness_local, int32_t P_local, int32_t k,
                            void* params, size_t param_bytes, int32_t* h_plan, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* POD_H */
