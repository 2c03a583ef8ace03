// Synchronized execution on the device: one lockstep block of W samplers.
//
//   executor.py:451-510 run_epoch_lockstep / barrier_action -> pq_act_step
//     batched_inference (executor.py:106-112)   -> F1..F4 GEMMs over the W current stacks
//     select_action (agent.py:53-66)           -> k_act_env: explore = random() < eps,
//                                                 integers(A) when exploring, else argmax
//                                                 with lowest-index ties, on sampler j's
//                                                 own PCG64 stream (executor.py:59-63)
//     _sampler_step (executor.py:237-249)      -> env.step on the same stream, transition
//                                                 record into the sampler buffer (staging),
//                                                 bootstrap terminal = terminal && !truncated,
//                                                 episode log, reset
//   epsilon_at (agent.py:44-50) is evaluated in fp64 with the reference formula.
// The environment is the synthetic frame env of oracle/envs.py (reward draw, terminal
// draw, counter-hashed 84x84 frames, 4-frame stack with masked history).
#include "../../include/paraq_b200.h"
#include "common.cuh"
#include "qnet.cuh"

namespace pq {
int set_err(const char *msg);
int cuda_err(cudaError_t e, const char *where);
int act_forward(pq_net net, const uint8_t *ring, const int32_t *stack, int W, int A, void *ws,
                int max_batch, const float **part_out, uint32_t **done_out, int *splits_out, cudaStream_t st);

__device__ __forceinline__ uint64_t env_frame_base(uint64_t key, int64_t episode, int t, int action) {
    return splitmix64(splitmix64(splitmix64(key) ^ (uint64_t)episode) ^
                      (((uint64_t)t << 8) | (uint64_t)action));
}

__device__ __forceinline__ double epsilon_at(int64_t t, double start, double end, int64_t anneal) {
    if (t >= anneal || anneal == 1) return end;
    double frac = (double)(t - 1) / (double)(anneal - 1);
    return __dadd_rn(start, __dmul_rn(__dsub_rn(end, start), frac));
}

struct ActArgs {
    const float *part;   // fc1 partials [S][W][512]
    const float *master;
    pq_envs e;
    uint8_t *ring;
    int32_t *staging;
    int32_t *step_counter;
    uint32_t *done;
    int W, steps, A, L;
    int sampler0, W_total;  // sharded acting: global index of sampler 0, samplers of the run
    int64_t epoch_start, frame_capacity;
    double eps_start, eps_end;
    int64_t eps_anneal;
    double term_p;
    float *q_out;
    int max_episodes;
    int splits;  // fc1 partial splits (FC1_SPLITS, or 1 after k_fc1_acc7)
};

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(256) k_act_env(const ActArgs a) {
    const int j = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    griddep_wait();
    griddep_launch();
    __shared__ float hs[512];
    __shared__ float qs[MAX_ACTIONS];
    __shared__ uint64_t s_base[2];
    __shared__ int64_t s_slot[2];
    // sampler state: every load issued up front by thread 0 (independent, in flight
    // together with the fc1 reduction below)
    uint64_t pcg[6] = {}, key = 0;
    int32_t st4[4] = {}, t0 = 0, epc = 0;
    int64_t ep0 = 0, seq = 0, bg = 0;
    double ret0 = 0.0;
    if (tid == 0) {
        bg = *a.step_counter;
#pragma unroll
        for (int k = 0; k < 6; ++k) pcg[k] = a.e.pcg[j * 6 + k];
        const int4 sv = *reinterpret_cast<const int4 *>(a.e.stack + j * 4);
        st4[0] = sv.x, st4[1] = sv.y, st4[2] = sv.z, st4[3] = sv.w;
        t0 = a.e.t[j];
        ep0 = a.e.episode[j];
        seq = a.e.slot_next[j];
        key = a.e.key[j];
        ret0 = a.e.ep_return[j];
        epc = a.e.ep_count[j];
    }
    {
        float v[2][FC1_SPLITS + 1];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int jj = tid + 256 * i;
#pragma unroll
            for (int sp = 0; sp < FC1_SPLITS; ++sp)
                v[i][sp] = sp < a.splits ? a.part[((size_t)sp * a.W + j) * 512 + jj] : 0.f;
            v[i][FC1_SPLITS] = a.master[P_B4 + jj];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float s = 0.f;
#pragma unroll
            for (int sp = 0; sp < FC1_SPLITS; ++sp)
                if (sp < a.splits) s += v[i][sp];
            s += v[i][FC1_SPLITS];
            hs[tid + 256 * i] = s > 0.f ? s : 0.f;
        }
    }
    __syncthreads();
    {
        float wv[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int aa = min(warp + 8 * u, a.A - 1);
#pragma unroll
            for (int t = 0; t < 16; ++t) wv[u][t] = a.master[P_W5 + aa * 512 + lane + 32 * t];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int aa = warp + 8 * u;
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 16; ++t) acc += wv[u][t] * hs[lane + 32 * t];
            acc = warp_sum_f(acc);
            if (lane == 0 && aa < a.A) {
                const float q = acc + a.master[p_b5(a.A) + aa];
                qs[aa] = q;
                if (a.q_out) a.q_out[j * a.A + aa] = q;
            }
        }
    }
    __shared__ bool s_active;
    const bool compact = a.e.reset_next != nullptr;
    if (tid == 0) {
        s_active = a.max_episodes <= 0 || epc < a.max_episodes;
        s_slot[0] = s_slot[1] = -1;
        if (compact) a.e.reset_ep[j] = -1;  // set below when this env resets
    }
    __syncthreads();
    if (tid == 0 && s_active) {
        // step_counter counts lockstep blocks (run-global in the executor); the
        // staging row is the block index within the epoch
        const int b = (int)(bg % a.steps);
        const int64_t t_label = a.epoch_start + bg * a.W_total + a.sampler0 + j + 1;
        const double eps = epsilon_at(t_label, a.eps_start, a.eps_end, a.eps_anneal);
        Pcg64 g;
        g.load(pcg);
        int act;
        if (g.random() < eps) {
            act = (int)g.bounded((uint32_t)a.A);
        } else {
            act = 0;
            for (int aa = 1; aa < a.A; ++aa)
                if (qs[aa] > qs[act]) act = aa;
        }
        // env.step(action, rng): reward draw, terminal draw, next frame
        const double reward = g.random();
        const bool term = g.random() < a.term_p;
        int t = t0 + 1;
        int64_t ep = ep0;
        const int32_t fs = (int32_t)(seq % a.frame_capacity);
        s_slot[0] = fs;
        s_base[0] = env_frame_base(key, ep, t, act);
        const bool trunc = !term && t >= a.L;
        int4 *rec = reinterpret_cast<int4 *>(a.staging + ((int64_t)j * a.steps + b) * REC_INTS);
        rec[0] = make_int4(st4[0], st4[1], st4[2], st4[3]);
        int32_t hi[3];
        rec_pack(hi, act, term, reward);
        rec[1] = make_int4(fs, hi[0], hi[1], hi[2]);
        double ret = ret0 + reward;
        s_slot[1] = -1;
        int4 nst;
        if (term || trunc) {
            if (epc < a.steps) {  // the episode log holds `steps` entries per sampler
                a.e.ep_label[(int64_t)j * a.steps + epc] = t_label;
                a.e.ep_ret[(int64_t)j * a.steps + epc] = ret;
            }
            a.e.ep_count[j] = epc + 1;
            ret = 0.0;
            ep += 1;
            t = 0;
            s_base[1] = env_frame_base(key, ep, 0, 255);
            if (compact) {  // slot assigned by the step's last CTA (below), frame written then
                s_slot[1] = -2;
                a.e.reset_ep[j] = ep;
                nst = make_int4(-1, -1, -1, -1);
                a.e.slot_next[j] = seq + 1;
            } else {
                const int32_t rs = (int32_t)((seq + 1) % a.frame_capacity);
                s_slot[1] = rs;
                nst = make_int4(-1, -1, -1, rs);
                a.e.slot_next[j] = seq + 2;
            }
        } else {
            nst = make_int4(st4[1], st4[2], st4[3], fs);
            a.e.slot_next[j] = seq + 1;
        }
        if (s_slot[1] != -2) *reinterpret_cast<int4 *>(a.e.stack + j * 4) = nst;
        a.e.ep_return[j] = ret;
        a.e.t[j] = t;
        a.e.episode[j] = ep;
        a.e.actions[j] = act;
        uint64_t out[6];
        g.store(out);
#pragma unroll
        for (int k = 0; k < 6; ++k) a.e.pcg[j * 6 + k] = out[k];
    }
    __syncthreads();
    for (int f = 0; f < 2 && s_active; ++f) {
        if (s_slot[f] < 0) continue;
        uint64_t *d = reinterpret_cast<uint64_t *>(a.ring + (size_t)s_slot[f] * FRAME_BYTES);
        for (int p = tid; p < FRAME_BYTES / 8; p += blockDim.x) d[p] = splitmix64(s_base[f] + (uint64_t)p);
    }
    // the last CTA advances the block counter (every CTA has read it by then)
    __shared__ bool s_last;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (compact && s_last) {  // reset-frame slots of this step, consecutive in sampler order
        __shared__ int s_wsum[8];
        __shared__ int64_t s_rn;
        __shared__ int s_tot;
        if (tid == 0) s_rn = *reinterpret_cast<volatile int64_t *>(a.e.reset_next), s_tot = 0;
        __syncthreads();
        for (int c0 = 0; c0 < a.W; c0 += 256) {
            const int jj = c0 + tid;
            const int64_t rep = jj < a.W ? *reinterpret_cast<volatile int64_t *>(a.e.reset_ep + jj) : -1;
            const bool f = rep >= 0;
            const unsigned m = __ballot_sync(0xffffffffu, f);
            if (lane == 0) s_wsum[warp] = __popc(m);
            __syncthreads();
            int before = s_tot;
            for (int w = 0; w < warp; ++w) before += s_wsum[w];
            if (f) {
                const int32_t rs = (int32_t)((s_rn + before + __popc(m & ((1u << lane) - 1u))) % a.frame_capacity);
                a.e.reset_slot[jj] = rs;
                *reinterpret_cast<int4 *>(a.e.stack + jj * 4) = make_int4(-1, -1, -1, rs);
            }
            __syncthreads();
            if (tid == 0)
                for (int w = 0; w < 8; ++w) s_tot += s_wsum[w];
            __syncthreads();
        }
        if (tid == 0) *a.e.reset_next = s_rn + s_tot;
    }
    if (s_last && tid == 0) {
        __threadfence();
        *reinterpret_cast<volatile int32_t *>(a.step_counter) = (int32_t)(bg + 1);
        *a.done = 0;
        __threadfence();
    }
    if (compact && s_slot[1] == -2) {
        // this env reset: wait for the last CTA's slot assignment (it has arrived, so it
        // is resident and runs to completion), then write the reset frame
        __shared__ int32_t s_rs;
        if (tid == 0) {
            if (!s_last)
                while (*reinterpret_cast<volatile int32_t *>(a.step_counter) == (int32_t)bg) __nanosleep(64);
            __threadfence();
            s_rs = *reinterpret_cast<volatile int32_t *>(a.e.reset_slot + j);
        }
        __syncthreads();
        uint64_t *d = reinterpret_cast<uint64_t *>(a.ring + (size_t)s_rs * FRAME_BYTES);
        for (int p = tid; p < FRAME_BYTES / 8; p += blockDim.x) d[p] = splitmix64(s_base[1] + (uint64_t)p);
    }
}

__global__ void k_env_reset(pq_envs e, int W, const int32_t *slots, uint8_t *ring) {
    const int j = blockIdx.x;
    __shared__ uint64_t base;
    if (threadIdx.x == 0) {
        int64_t ep = e.episode[j] + 1;
        e.episode[j] = ep;
        e.t[j] = 0;
        e.ep_return[j] = 0.0;
        int32_t *st4 = e.stack + j * 4;
        st4[0] = st4[1] = st4[2] = -1;
        st4[3] = slots[j];
        base = env_frame_base(e.key[j], ep, 0, 255);
    }
    __syncthreads();
    uint64_t *d = reinterpret_cast<uint64_t *>(ring + (size_t)slots[j] * FRAME_BYTES);
    for (int p = threadIdx.x; p < FRAME_BYTES / 8; p += blockDim.x) d[p] = splitmix64(base + (uint64_t)p);
}

}  // namespace pq

using namespace pq;

extern "C" {

int pq_env_reset(pq_envs envs, int W, const int32_t *slots, uint8_t *ring, void *stream) {
    if (W <= 0) return 0;
    k_env_reset<<<W, 128, 0, (cudaStream_t)stream>>>(envs, W, slots, ring);
    return cuda_err(cudaGetLastError(), "env_reset");
}

int pq_act_step(const pq_act_args *x, void *stream) {
    if (x->W < 1 || x->W > x->max_batch) return set_err("W out of range for the workspace");
    if (x->actions < 1 || x->actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    cudaStream_t st = (cudaStream_t)stream;
    const float *part = nullptr;
    uint32_t *done = nullptr;
    int splits = FC1_SPLITS;
    int rc = act_forward(x->net, x->ring, x->envs.stack, x->W, x->actions, x->ws, x->max_batch,
                         &part, &done, &splits, st);
    if (rc) return rc;
    ActArgs a{};
    a.part = part;
    a.master = x->net.master;
    a.e = x->envs;
    a.ring = x->ring;
    a.staging = x->staging;
    a.step_counter = x->step_counter;
    a.done = done;
    a.W = x->W, a.steps = x->steps, a.A = x->actions, a.L = x->episode_length;
    a.sampler0 = x->sampler0, a.W_total = x->W_total > 0 ? x->W_total : x->W;
    a.epoch_start = x->epoch_start;
    a.frame_capacity = x->frame_capacity;
    a.eps_start = x->eps_start, a.eps_end = x->eps_end, a.eps_anneal = x->eps_anneal;
    a.term_p = x->terminal_p;
    a.q_out = x->q_out;
    a.max_episodes = x->max_episodes;
    a.splits = splits;
    return cuda_err(launch_k(k_act_env, dim3(x->W), dim3(256), 0, st, a), "act_env");
}

}  // extern "C"
