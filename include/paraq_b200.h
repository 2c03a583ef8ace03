/*
 * paraq_b200.h -- C ABI of the B200-native fast-DQN hot path
 * (arXiv 2111.01264: concurrent training + synchronized execution).
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t passed
 * as void*, returns 0 on success and a nonzero status on error (pq_last_error()
 * gives the message; the Python shim maps it to ValueError / RuntimeError like
 * the reference).  No torch types cross this boundary.  All kernels are sm_100a.
 *
 * Reference interfaces each group replaces (paths under /root/reference/pkg/src/paraq):
 *   replay sampling ..... replay.py:61-66   ReplayMemory.sample -> rng.integers(0, len, B)
 *   replay flush ........ replay.py:82-93   ReplayMemory.flush (owner-major order)
 *   prepopulation ....... replay.py:68-80   ReplayMemory.prepopulate
 *   batch gather ........ agent.py:76,:100  np.stack of states / next states
 *   Q forward ........... nn.py:123-131     forward  (kernels affine_rows/relu, _kernels_numba.py:19-42)
 *   learner step ........ agent.py:84-105   train_minibatch = td_targets (agent.py:69-81)
 *                                           + gradient (nn.py:134-170) + rmsprop_step (nn.py:173-203)
 *   acting .............. executor.py:106-112 batched_inference + agent.py:53-66 select_action
 *                                           + executor.py:237-249 _sampler_step
 *   target sync ......... nn.py:206-211     copy_parameters (executor.py:559)
 *   theta hash .......... nn.py:214-229     parameter_bytes + theta_hash (FNV-1a 64)
 *   kernel plugin ....... backend.py:18-34 / _kernels_numba.py:19-111 (fp64 kernel module)
 */
#ifndef PARAQ_B200_H
#define PARAQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQ_ABI_VERSION 1
#define PQ_FRAME_BYTES 7056 /* one 84x84 uint8 frame */
#define PQ_REC_INTS 8       /* replay record: frame slots f0..f4, action | terminal << 16,
                               reward as f64 bits (lo, hi) */

/* ---- housekeeping ---------------------------------------------------------- */
int pq_abi_version(void);
const char *pq_last_error(void);
int64_t pq_num_params(int actions);          /* 1,693,362 for 18 actions */
int64_t pq_num_shadow(void);                 /* bf16 copies of the conv1..fc1 weights */
/* Latency probes: enable/disable and read GEMM phase timestamps (out [256][12] ns). */
int pq_timeline(int on, unsigned long long *out, int *count);
int pq_timeline_tma(int on, unsigned long long *out, int *count); /* the TMA-engine kernels' probes */
/* Per-CTA trace of the learner kernels: out [8192][6] = start, dependency released,
 * accumulator ready, end (ns), smid << 32 | linear CTA, tag << 48 | part << 40 | grid. */
int pq_cta_trace(int on, unsigned long long *out, int *count);
/* A cudaStream_t (as void*) on a green-context partition of >= sm_count SMs (multiples of
 * 8 on sm_100a; *sm_granted = the partition's size): the executor's acting stream under
 * PQ_ACT_SMS, so lockstep acting blocks stay off the SMs the learner grids use.  No
 * reference counterpart (the reference's samplers are CPU threads). */
int pq_sm_partition_stream(int sm_count, void **stream_out, int *sm_granted);

/* ---- one Q-network parameter set (theta or theta-minus), device memory ------------ */
typedef struct pq_net {
    float *master;     /* fp32 [pq_num_params] in nn.parameter_bytes order */
    uint16_t *shadow;  /* bf16 [pq_num_shadow] GEMM copies of W1..W4 */
} pq_net;

typedef struct pq_opt {
    float *m; /* first moments  (nn.OptState.m_*) */
    float *v; /* second moments (nn.OptState.v_*) */
} pq_opt;

/* Refresh the bf16 shadow from the fp32 master (after an upload). */
int pq_net_sync_shadow(pq_net net, void *stream);
/* theta-minus <- theta (copy_parameters, nn.py:206-211; executor.py:559) */
int pq_net_copy(pq_net dst, pq_net src, int actions, void *stream);
/* L2 residency of the learner's working set: kernels launched into `stream` (and graph
 * kernel nodes captured from it) keep [base, base + bytes) in the persisting L2 set-aside
 * (hit_ratio of its lines, capped to the set-aside); bytes = 0 clears the window. */
int pq_l2_persist(void *stream, const void *base, size_t bytes, float hit_ratio);

/* ---- frame-stack addressing -------------------------------------------------------
 * A state is 4 frames; frames live in a uint8 ring [slots][7056].  Sample b,
 * channel c reads slot refs[map(b) * ref_stride + ref_off + c] (map = identity when
 * NULL); slot -1 is the all-zero (masked) frame.  Replay records [cap][8] int32 are
 * {f0, f1, f2, f3, f4, action | terminal << 16, reward_lo, reward_hi} (terminal = the
 * bootstrap terminal, executor.py:241; reward = the f64 bits of the reference's float):
 * state = (f0..f3), next state = (f1..f4), so ref_off 0 / 1 selects s / s'. */

/* ---- replay (replay.py) ----------------------------------------------------------- */
/* rng.integers(0, n, size=count), bit-exact with numpy PCG64 + buffered Lemire;
 * pcg_state: device u64[6] {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger},
 * updated in place.  1 <= n < 2^32. */
int pq_sample_indices(uint64_t *pcg_state, uint32_t n, int64_t count, int64_t *idx_out,
                      void *stream);
/* Stack gather of a sampled batch: s_out / s2_out [B][4][84][84] uint8,
 * a_out int32 [B], r_out f64 [B], term_out uint8 [B]. */
int pq_replay_gather(const uint8_t *ring, const int32_t *records, const int64_t *idx,
                     int64_t B, uint8_t *s_out, uint8_t *s2_out, int32_t *a_out, double *r_out,
                     uint8_t *term_out, void *stream);
/* the two engines behind pq_replay_gather (default: 16-byte vector loads; PQ_GATHER=tma
 * selects TMA bulk copies of whole frames through a shared-memory ring) */
int pq_replay_gather_tma(const uint8_t *ring, const int32_t *records, const int64_t *idx,
                     int64_t B, uint8_t *s_out, uint8_t *s2_out, int32_t *a_out, double *r_out,
                     uint8_t *term_out, void *stream);
int pq_replay_gather_ldg(const uint8_t *ring, const int32_t *records, const int64_t *idx,
                     int64_t B, uint8_t *s_out, uint8_t *s2_out, int32_t *a_out, double *r_out,
                     uint8_t *term_out, void *stream);
/* Flush: staging records [W][steps][8] -> ring records in owner-major order,
 * slot = (push_count + j * steps + k) mod capacity. */
int pq_replay_flush(const int32_t *staging, int W, int steps, int32_t *records,
                    int64_t capacity, int64_t push_count, void *stream);
/* The same for the staged steps [k0, k1) of every sampler (the blocking training
 * event of the non-concurrent modes flushes mid-epoch, executor.py:436-440):
 * slot = (push_count + j * (k1 - k0) + k - k0) mod capacity. */
int pq_replay_flush_range(const int32_t *staging, int W, int steps, int k0, int k1,
                          int32_t *records, int64_t capacity, int64_t push_count, void *stream);

/* ---- synthetic frame environments (caller side, oracle/envs.py on the CPU) -------- */
typedef struct pq_envs {
    uint64_t *pcg;       /* [W][6] per-sampler PCG64 streams (executor.py:59-63) */
    int64_t *episode;    /* [W] episode index */
    int32_t *t;          /* [W] steps into the episode */
    int32_t *stack;      /* [W][4] frame slots of the current state (-1 = masked) */
    double *ep_return;   /* [W] running return */
    uint64_t *key;       /* [W] frame-hash key */
    int64_t *slot_next;  /* [W] next frame sequence number of this env (slot = seq mod ring size) */
    int32_t *ep_count;   /* [W] episodes finished this epoch */
    int64_t *ep_label;   /* [W][steps] t_label of finished episodes */
    double *ep_ret;      /* [W][steps] their returns */
    int32_t *actions;    /* [W] last actions (read back by the host API) */
    /* Optional compact frame allocation (NULL: each env takes seq + 1 for a reset frame,
     * i.e. 2 slots per step reserved).  Non-NULL: next frames take slot_next (1 per step)
     * and the reset frames of a step get consecutive sequence numbers from *reset_next in
     * sampler order, assigned by the step's last CTA (deterministic). */
    int64_t *reset_next; /* [1] next reset-frame sequence number */
    int64_t *reset_ep;   /* [W] scratch: new episode index of a resetting env, else -1 */
    int32_t *reset_slot; /* [W] scratch: assigned reset-frame slot */
} pq_envs;

/* Reset env j into frame slot slots[j] (episode start, masked stack). */
int pq_env_reset(pq_envs envs, int W, const int32_t *slots, uint8_t *ring, void *stream);

/* Prepopulation (replay.py:68-80) of n transitions from one env on the PREPOP
 * stream: frames into ring slots [frame_base, frame_base + used), records into
 * rec_out[n][8]; *frames_used_out (device int64) receives the slot count. */
int pq_prepopulate(uint64_t *pcg_state, uint64_t key, int episode_length, int actions,
                   double terminal_p, int64_t n, uint8_t *ring, int64_t frame_base,
                   int64_t frame_capacity, int32_t *rec_out, int64_t *frames_used_out,
                   void *scratch, void *stream);
/* The same in two calls, so the host can reserve exactly the frames the walk used
 * before any is written: the walk (records, frame descriptors in scratch, count), then
 * the frame generation into ring slots [frame_base, frame_base + *frames_used). */
int pq_prepopulate_walk(uint64_t *pcg_state, int episode_length, int actions, double terminal_p,
                        int64_t n, int64_t frame_base, int64_t frame_capacity, int32_t *rec_out,
                        int64_t *frames_used_out, void *scratch, void *stream);
int pq_prepopulate_frames(uint64_t key, uint8_t *ring, int64_t frame_base, int64_t frame_capacity,
                          const int64_t *frames_used, const void *scratch, void *stream);
size_t pq_prepopulate_scratch_bytes(int64_t n);

/* ---- Q network (nn.py / agent.py) -------------------------------------------------- */
size_t pq_workspace_bytes(int max_batch, int actions);
/* fc1 split-K partial slots the forward of `groups` networks (2: the learner's online +
 * target, 1: acting) leaves in the workspace at batch n (7, or 1 when the large-batch
 * kernel reduces the splits in TMEM; the head / acting kernels read that many). */
int pq_fc1_splits(int n, int groups);
/* Byte offsets of the workspace buffers (stage-wise kernel tests), in order:
 * act1, act2, act3, fc1part (online), act1, act2, act3, fc1part (target), q, h1, dh1,
 * td, dh1_bf16, dh1T_bf16, actions, dY3, dY2, dY1, part1, part2, part3, grad4, then dY1
 * on the padded 21 x 21 grid, dY2 on the padded 11 x 11 grid, act1 (online, target) as
 * 2x2 space-to-depth [n][10][10][128] (-1 below batch 128; the TMA engine's
 * shifted-descriptor conv kernels, which then leave the dense act1 unwritten). */
int pq_workspace_layout(int max_batch, int actions, int64_t *offsets);

/* Q-values for n states (nn.forward): q_out f32 [n][actions]. */
int pq_forward(pq_net net, const uint8_t *ring, const int32_t *refs, const int64_t *map,
               int ref_stride, int ref_off, int n, int actions, float *q_out, void *ws,
               int max_batch, void *stream);

typedef struct pq_learn_args {
    pq_net theta;          /* read */
    pq_opt opt;            /* read */
    pq_net theta_out;      /* written (may alias theta: elementwise update) */
    pq_opt opt_out;        /* written (may alias opt) */
    pq_net target;         /* theta-minus, read */
    const uint8_t *ring;
    const int32_t *records;
    const int64_t *idx;          /* [n] sampled record slots; NULL -> idx_base + counter */
    const int64_t *idx_base;     /* epoch index table, sliced by *update_counter */
    int32_t *update_counter;     /* device counter, incremented per step (graph replay) */
    const float *ext_targets;    /* optional: fixed targets (nn.gradient), skips the TD head */
    const int32_t *ext_actions;
    int n, actions;
    float gamma, lr, rho, kappa;
    int32_t *nonfinite;          /* device int: min update id with a non-finite gradient */
    float *grad_out;             /* optional f32 [num_params]: summed gradient */
    float *q_out;                /* optional f32 [2][n][actions]: online / target Q */
    float *td_out;               /* optional f32 [n][3]: target, delta, loss */
    void *ws;
    int max_batch;
    float huber;                 /* > 0: Huber TD loss with this delta (north star; opt-in);
                                    0 / inf: the reference's half-squared loss (nn.py:140-144) */
} pq_learn_args;

/* One learner step (agent.train_minibatch): target forward + max, online forward,
 * TD error, backward, centered RMSProp on the summed gradient. */
int pq_learn_step(const pq_learn_args *args, void *stream);
/* The same step with the target network's forward pipelined: step k's backward launches
 * also run the target conv1..conv3 of the minibatch at *update_counter + 1 and the next
 * step's conv1 launch its fc1 (theta-minus is fixed within an epoch).  Requires the
 * epoch-table mode (idx_base + update_counter, one spare table row), no external targets
 * and the small-batch fused schedule; otherwise identical to pq_learn_step.  Results are
 * bit-identical to pq_learn_step.  pq_learn_target_prologue computes the target
 * conv1..conv3 of the step at *update_counter (call it at the start of every epoch).
 * *update_counter advances inside the step's fc1 data-gradient launch (pq_learn_step:
 * at the end of its head), so only launches after the step may read it. */
int pq_learn_step_pipelined(const pq_learn_args *args, void *stream);
int pq_learn_target_prologue(const pq_learn_args *args, void *stream);

/* Data-parallel learner (configs[4]): the summed gradient of this
 * rank's shard of the batch (same forward / TD / backward as pq_learn_step, no update)
 * into grad f32 [pq_num_params]; the ranks sum-all-reduce it (NCCL) and every rank
 * applies the identical centered RMSProp with pq_rmsprop_apply (theta / opt in place,
 * bf16 shadow refreshed, *nonfinite = min(update_id) on a non-finite gradient).
 * agent.py:103-104 feeds the optimizer the summed gradient, so a sum of shard sums is
 * the reference semantics (fp32 summation order aside). */
int pq_learn_grad(const pq_learn_args *args, float *grad, void *stream);
/* The same, recording the cudaEvent_t fc1_done once grad[P_W4, P_B4) (the fc1 weight
 * gradient, 6.4 of the 6.77 MB) is complete: its all-reduce overlaps the conv backward. */
int pq_learn_grad_ev(const pq_learn_args *args, float *grad, void *stream, void *fc1_done);
int pq_rmsprop_apply(pq_net theta, pq_opt opt, const float *grad, int actions, float lr, float rho,
                     float kappa, int32_t *nonfinite, int update_id, void *stream);

typedef struct pq_act_args {
    pq_net net;                 /* acting parameters (theta-minus when concurrent) */
    pq_envs envs;
    uint8_t *ring;
    int32_t *staging;           /* [W][steps][8] transition records of this epoch */
    int32_t *step_counter;      /* device block counter bg: t_label = epoch_start + bg*W + j + 1,
                                   staging row = bg mod steps; incremented per call */
    int W, steps, actions, episode_length;
    int64_t epoch_start;        /* global step at the epoch start (t labels) */
    int64_t frame_capacity;     /* frame ring slots */
    double eps_start, eps_end;
    int64_t eps_anneal;
    double terminal_p;
    float *q_out;               /* optional [W][actions] */
    void *ws;
    int max_batch;
    int max_episodes;           /* > 0: a sampler stops after this many finished episodes
                                   (evaluate_policy's exact episode budget) */
    int sampler0;               /* global index of this launch's first sampler (sharded acting) */
    int W_total;                /* samplers of the whole run (t labels); 0 = W */
} pq_act_args;

/* One synchronized block (executor.py:451-510): batched Q inference for the W current
 * states, epsilon-greedy per sampler on its own PCG64 stream (agent.py:53-66), env
 * step, transition record into staging, episode bookkeeping and reset. */
int pq_act_step(const pq_act_args *args, void *stream);

/* ---- host-side samplers (end-to-end path: CPU envs, GPU inference) ---------------- */
typedef struct pq_henv {
    uint64_t pcg[6];   /* the sampler's PCG64 stream (shared by select_action and env.step) */
    uint64_t key;      /* frame-hash key */
    int64_t episode;
    int32_t t, pad;
    double ep_return;
} pq_henv;

int pq_henv_reset(pq_henv *envs, int W, int64_t *seq, int64_t frame_capacity, uint8_t *frames_out,
                  int32_t *stacks);
int pq_henv_step(pq_henv *envs, int W, const float *q, int A, int episode_length,
                 double terminal_p, int64_t t_label0, double eps_start, double eps_end,
                 int64_t eps_anneal, int64_t *seq, int64_t frame_capacity, uint8_t *frames_out,
                 int *nframes, int32_t *stacks, int32_t *records, int64_t *ep_labels,
                 double *ep_rets, int *n_eps);

/* ---- elementwise kernels of the reference kernel module (fp32 / fp64) ------------- */
int pq_rmsprop_f32(const float *p, const float *g, const float *m, const float *v, int64_t n,
                   float lr, float rho, float kappa, float *p2, float *m2, float *v2,
                   int32_t *nonfinite, void *stream);

/* ---- fp64 kernel module: the reference plugin API, bit-exact with numba ------------
 * _kernels_numba.py:19-111 (selected by backend.py:18-34); device pointers, float64,
 * C-contiguous, output buffers caller-allocated. */
int pq64_affine_rows(const double *w, const double *b, const double *x, int64_t n, int64_t o,
                     int64_t d, double *out, void *stream);
int pq64_relu(const double *x, int64_t count, double *out, void *stream);
int pq64_output_delta(const double *q, const int64_t *actions, const double *targets, int64_t n,
                      int64_t o, double *delta, void *stream);
int pq64_weight_grad(const double *delta, const double *acts, int64_t n, int64_t o, int64_t d,
                     double *dw, void *stream);
int pq64_bias_grad(const double *delta, int64_t n, int64_t o, double *db, void *stream);
int pq64_hidden_delta(const double *delta, const double *w, const double *pre, int64_t n,
                      int64_t o, int64_t d, double *out, void *stream);
int pq64_rmsprop_flat(const double *p, const double *g, const double *m, const double *v,
                      int64_t count, double lr, double rho, double kappa, double *p2, double *m2,
                      double *v2, void *stream);

/* ---- host-side helpers ---------------------------------------------------------- */
/* theta_hash (nn.py:223-229): FNV-1a 64 over the little-endian float64 bytes of the
 * parameters (fp32 master widened to f64), layer order weights then bias. */
uint64_t pq_theta_hash_f32(const float *host_params, int64_t n);
uint64_t pq_theta_hash_f64(const double *host_params, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* PARAQ_B200_H */
