// Non-GEMM pieces of the learner step, as device functions shared by the one-shot
// kernels (qnet.cu: k_head, k_optimizer) and the persistent learner (learner.cu).
//
//   head_sample  -- fc1 split-K reduction + bias + ReLU, fc2, and for the learner the TD
//                   target (agent.py:69-81: r if terminal else r + gamma * max_a Q-(s')),
//                   the output delta (nn.py:137-144 output_delta, summed-gradient
//                   convention of agent.py:103-104) and its back-prop through fc2 and
//                   the fc1 ReLU mask (hidden_delta, _kernels_numba.py:80-95).
//   opt_param    -- one parameter of the centered RMSProp step (_kernels_numba.py:98-111,
//                   kappa inside the square root) on the summed gradient, reducing the
//                   split-K weight-gradient partials in a fixed order; refreshes the bf16
//                   GEMM shadow and raises the non-finite flag (nn.py:181-183).
//
// Loads are plain ld.global: data written earlier in a persistent launch is visible
// because the grid barrier's gpu-scope fences invalidate the SM's L1 (CCTL.IVALL);
// never the non-coherent path.
#pragma once

#include "gemm.cuh"
#include "qnet.cuh"

namespace pq {

struct HeadArgs {
    const float *part[2];  // fc1 split-K partials [splits][n][512] of group 0 / 1
    const float *master[2];
    int groups, n, A, n8;
    int splits;  // fc1 partial splits to sum (FC1_SPLITS, or 1 after k_fc1_acc7)
    int block;   // samples per CTA (1: head_sample; HEAD_BLOCK: head_block, with splits == 1)
    const int32_t *records;
    const int64_t *idx;       // sampled slots, or
    const int64_t *idx_base;  // epoch table sliced by *counter
    const int32_t *counter;
    const float *ext_targets;
    const int32_t *ext_actions;
    float gamma;
    float huber;  // > 0: Huber TD loss with this delta (dL/dq clipped to [-huber, huber])
    int learner;
    float *q_out;  // [groups][n][A]
    float *h1, *dh1, *td;
    bf16 *dh1_bf, *dh1T;
    int32_t *act_out;
    float *q_copy;   // optional extra copy [groups][n][A]
    float *td_copy;  // optional [n][3]
    int64_t *idx_cur;  // optional: the step's sampled slots [n] (read later without the counter)
    int32_t *upd_cur;  // optional: the step's update id (*counter before the bump)
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int HEAD_THREADS = 256;
constexpr int HEAD_BLOCK = 4;  // samples per head CTA at large batches

// One sample b (one 256-thread CTA).  S = fc1 split count; every global load of a
// phase is independent so they are all in flight together.  Everything that does not
// depend on the fc1 forward -- the sampled record, the fc1 / fc2 biases, the fc2
// weights (prefetched into L1) -- is requested before `wait()` (the kernel's
// griddepcontrol.wait): they were written four or more launches back.
template <int S, class Wait = NoHook>
PQ_DEV void head_sample(const HeadArgs &a, int b, Wait wait = Wait{}) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ float hs[2][512];
    __shared__ float qs[2][MAX_ACTIONS];
    __shared__ float s_delta;
    __shared__ int s_act;
    // the sampled record (action, reward, terminal) is fetched early by thread 0
    int4 rec_hi = make_int4(0, 0, 0, 0);
    if (a.learner && tid == 0) {
        int64_t slot = a.idx        ? a.idx[b]
                       : a.idx_base ? a.idx_base[(int64_t)(*a.counter) * a.n + b]
                                    : (int64_t)b;
        if (!a.ext_targets) rec_hi = *reinterpret_cast<const int4 *>(a.records + slot * REC_INTS + 4);
        if (a.idx_cur) a.idx_cur[b] = slot;
        if (a.upd_cur && b == 0) *a.upd_cur = a.counter ? *a.counter : 0;
    }
    float b4[2][2], b5[2][4];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const int gg = g < a.groups ? g : 0;
#pragma unroll
        for (int i = 0; i < 2; ++i) b4[g][i] = (*(a.master[gg] + P_B4 + tid + HEAD_THREADS * i));
#pragma unroll
        for (int u = 0; u < 4; ++u) b5[g][u] = (*(a.master[gg] + p_b5(a.A) + min(warp + 8 * u, a.A - 1)));
        // fc2 weights: A x 512 floats = A x 16 lines of 128 B per network
        for (int l = tid; l < a.A * 16; l += HEAD_THREADS)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.master[gg] + P_W5 + l * 32));
    }
    wait();
    {
        float v[2][2][S + 1];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = tid + HEAD_THREADS * i;
                const int gg = g < a.groups ? g : 0;
                const float *P = a.part[gg] + (size_t)b * 512 + j;
#pragma unroll
                for (int sp = 0; sp < S; ++sp) v[g][i][sp] = (*(P + (size_t)sp * a.n * 512));
                v[g][i][S] = b4[g][i];
            }
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                float s = 0.f;
#pragma unroll
                for (int sp = 0; sp < S; ++sp) s += v[g][i][sp];
                s += v[g][i][S];
                hs[g][tid + HEAD_THREADS * i] = s > 0.f ? s : 0.f;
            }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        if (g >= a.groups) break;
        const float *w5 = a.master[g] + P_W5;
        float wv[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int aa = min(warp + 8 * u, a.A - 1);
#pragma unroll
            for (int t = 0; t < 16; ++t) wv[u][t] = (*(w5 + aa * 512 + lane + 32 * t));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int aa = warp + 8 * u;
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 16; ++t) acc += wv[u][t] * hs[g][lane + 32 * t];
            acc = warp_sum(acc);
            if (lane == 0 && aa < a.A) {
                float q = acc + b5[g][u];
                qs[g][aa] = q;
                a.q_out[((size_t)g * a.n + b) * a.A + aa] = q;
                if (a.q_copy) a.q_copy[((size_t)g * a.n + b) * a.A + aa] = q;
            }
        }
    }
    if (!a.learner) return;
    __syncthreads();
    if (tid == 0) {
        int act;
        float target;
        if (a.ext_targets) {
            act = a.ext_actions[b];
            target = a.ext_targets[b];
        } else {
            act = rec_action(rec_hi.y);
            // td_targets (agent.py:69-81) in f64 on the f64 reward, rounded once
            const double r = rec_reward(rec_hi.z, rec_hi.w);
            if (rec_terminal(rec_hi.y)) {
                target = (float)r;
            } else {
                float mx = qs[1][0];
                for (int aa = 1; aa < a.A; ++aa) mx = fmaxf(mx, qs[1][aa]);
                target = (float)(r + (double)a.gamma * (double)mx);
            }
        }
        const float e = qs[0][act] - target;
        // d = n * output_delta (agent.py:103-104 summed gradient); the opt-in Huber loss
        // clips it (huber <= 0 or inf: the reference's half-squared loss)
        float d = e, loss = 0.5f * e * e;
        if (a.huber > 0.f && fabsf(e) > a.huber) {
            d = copysignf(a.huber, e);
            loss = a.huber * (fabsf(e) - 0.5f * a.huber);
        }
        s_delta = d;
        s_act = act;
        a.act_out[b] = act;
        a.td[b * 3 + 0] = target;
        a.td[b * 3 + 1] = d;
        a.td[b * 3 + 2] = loss;
        if (a.td_copy) {
            a.td_copy[b * 3 + 0] = target;
            a.td_copy[b * 3 + 1] = d;
            a.td_copy[b * 3 + 2] = loss;
        }
    }
    __syncthreads();
    const float d = s_delta;
    const float *w5 = a.master[0] + P_W5 + (size_t)s_act * 512;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int j = tid + HEAD_THREADS * i;
        const float hv = hs[0][j];
        const float g = hv > 0.f ? d * (*(w5 + j)) : 0.f;  // hidden_delta with the fc1 ReLU mask
        a.h1[(size_t)b * 512 + j] = hv;
        a.dh1[(size_t)b * 512 + j] = g;
        const bf16 gb = __float2bfloat16_rn(g);
        a.dh1_bf[(size_t)b * 512 + j] = gb;
        a.dh1T[(size_t)j * a.n8 + b] = gb;
    }
}

// NB samples per CTA (large batches, fc1 splits reduced by the forward: S = 1): the fc2
// weights (A x 512 per network) are read once per NB samples instead of once per sample,
// and the transposed bf16 hidden gradient goes out as NB contiguous values per unit.
// Per sample the arithmetic is head_sample's, operation for operation.
template <int S, int NB, class Wait = NoHook>
PQ_DEV void head_block(const HeadArgs &a, int b0, Wait wait = Wait{}) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nb = min(NB, a.n - b0);
    __shared__ float hs[NB][2][512];
    __shared__ float qs[NB][2][MAX_ACTIONS];
    __shared__ float s_delta[NB];
    __shared__ int s_act[NB];
    int4 rec_hi = make_int4(0, 0, 0, 0);  // thread s < nb: sample b0 + s
    if (a.learner && tid < nb) {
        const int b = b0 + tid;
        int64_t slot = a.idx        ? a.idx[b]
                       : a.idx_base ? a.idx_base[(int64_t)(*a.counter) * a.n + b]
                                    : (int64_t)b;
        if (!a.ext_targets) rec_hi = *reinterpret_cast<const int4 *>(a.records + slot * REC_INTS + 4);
        if (a.idx_cur) a.idx_cur[b] = slot;
        if (a.upd_cur && b == 0) *a.upd_cur = a.counter ? *a.counter : 0;
    }
    float b4[2][2], b5[2][4];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const int gg = g < a.groups ? g : 0;
#pragma unroll
        for (int i = 0; i < 2; ++i) b4[g][i] = (*(a.master[gg] + P_B4 + tid + HEAD_THREADS * i));
#pragma unroll
        for (int u = 0; u < 4; ++u) b5[g][u] = (*(a.master[gg] + p_b5(a.A) + min(warp + 8 * u, a.A - 1)));
        for (int l = tid; l < a.A * 16; l += HEAD_THREADS)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.master[gg] + P_W5 + l * 32));
    }
    wait();
#pragma unroll
    for (int sb = 0; sb < NB; ++sb) {
        if (sb >= nb) break;
        const int b = b0 + sb;
        float v[2][2][S + 1];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = tid + HEAD_THREADS * i;
                const int gg = g < a.groups ? g : 0;
                const float *P = a.part[gg] + (size_t)b * 512 + j;
#pragma unroll
                for (int sp = 0; sp < S; ++sp) v[g][i][sp] = (*(P + (size_t)sp * a.n * 512));
                v[g][i][S] = b4[g][i];
            }
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                float s = 0.f;
#pragma unroll
                for (int sp = 0; sp < S; ++sp) s += v[g][i][sp];
                s += v[g][i][S];
                hs[sb][g][tid + HEAD_THREADS * i] = s > 0.f ? s : 0.f;
            }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        if (g >= a.groups) break;
        const float *w5 = a.master[g] + P_W5;
        float wv[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int aa = min(warp + 8 * u, a.A - 1);
#pragma unroll
            for (int t = 0; t < 16; ++t) wv[u][t] = (*(w5 + aa * 512 + lane + 32 * t));
        }
#pragma unroll 1
        for (int sb = 0; sb < nb; ++sb) {
            const int b = b0 + sb;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int aa = warp + 8 * u;
                float acc = 0.f;
#pragma unroll
                for (int t = 0; t < 16; ++t) acc += wv[u][t] * hs[sb][g][lane + 32 * t];
                acc = warp_sum(acc);
                if (lane == 0 && aa < a.A) {
                    float q = acc + b5[g][u];
                    qs[sb][g][aa] = q;
                    a.q_out[((size_t)g * a.n + b) * a.A + aa] = q;
                    if (a.q_copy) a.q_copy[((size_t)g * a.n + b) * a.A + aa] = q;
                }
            }
        }
    }
    if (!a.learner) return;
    __syncthreads();
    if (tid < nb) {
        const int sb = tid, b = b0 + sb;
        int act;
        float target;
        if (a.ext_targets) {
            act = a.ext_actions[b];
            target = a.ext_targets[b];
        } else {
            act = rec_action(rec_hi.y);
            const double r = rec_reward(rec_hi.z, rec_hi.w);
            if (rec_terminal(rec_hi.y)) {
                target = (float)r;
            } else {
                float mx = qs[sb][1][0];
                for (int aa = 1; aa < a.A; ++aa) mx = fmaxf(mx, qs[sb][1][aa]);
                target = (float)(r + (double)a.gamma * (double)mx);
            }
        }
        const float e = qs[sb][0][act] - target;
        float d = e, loss = 0.5f * e * e;
        if (a.huber > 0.f && fabsf(e) > a.huber) {
            d = copysignf(a.huber, e);
            loss = a.huber * (fabsf(e) - 0.5f * a.huber);
        }
        s_delta[sb] = d;
        s_act[sb] = act;
        a.act_out[b] = act;
        a.td[b * 3 + 0] = target;
        a.td[b * 3 + 1] = d;
        a.td[b * 3 + 2] = loss;
        if (a.td_copy) {
            a.td_copy[b * 3 + 0] = target;
            a.td_copy[b * 3 + 1] = d;
            a.td_copy[b * 3 + 2] = loss;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int j = tid + HEAD_THREADS * i;
        bf16 gbs[NB];
#pragma unroll
        for (int sb = 0; sb < NB; ++sb) {
            gbs[sb] = __float2bfloat16_rn(0.f);
            if (sb >= nb) continue;
            const int b = b0 + sb;
            const float d = s_delta[sb];
            const float hv = hs[sb][0][j];
            const float g = hv > 0.f ? d * (*(a.master[0] + P_W5 + (size_t)s_act[sb] * 512 + j)) : 0.f;
            a.h1[(size_t)b * 512 + j] = hv;
            a.dh1[(size_t)b * 512 + j] = g;
            gbs[sb] = __float2bfloat16_rn(g);
            a.dh1_bf[(size_t)b * 512 + j] = gbs[sb];
        }
        bf16 *dT = a.dh1T + (size_t)j * a.n8 + b0;
        if (NB == 8 && nb == 8 && ((reinterpret_cast<uintptr_t>(dT) & 15) == 0)) {
            *reinterpret_cast<uint4 *>(dT) = *reinterpret_cast<const uint4 *>(gbs);
        } else if (NB == 4 && nb == 4 && ((reinterpret_cast<uintptr_t>(dT) & 7) == 0)) {
            *reinterpret_cast<uint2 *>(dT) = *reinterpret_cast<const uint2 *>(gbs);
        } else {
            for (int sb = 0; sb < nb; ++sb) dT[sb] = gbs[sb];
        }
    }
}

// ------------------------------------------------------------------ optimizer
struct OptArgs {
    const float *p, *m, *v;
    float *p2, *m2, *v2;
    bf16 *shadow;
    const float *part1, *part2, *part3, *grad4;
    int s1, s2, s3;
    const float *dh1, *h1, *td;
    const int32_t *act;
    int n, A;
    float lr, rho, kappa;
    int32_t *flag;
    int32_t *counter;  // update id source (read only)
    uint32_t *done;
    float *grad_out;
    int64_t total;
    int64_t lo1, hi1, lo2, hi2;  // k_optimizer: the parameter ranges it updates
    int32_t *bump;               // optional: step counter the last CTA advances
    uint32_t *bump_done;         // CTA completion counter for that increment
    const float *fcpart;         // optional: per-64-sample-chunk partials [chunks][A+2][512] of
    int fcchunks;                //   the fc2 / fc1-bias batch sums (k_fc2_partials)
    int w1_perm;                 // part1 rows in the permuted conv1 K order (TMA conv1 wgrad)
};

__device__ __forceinline__ float sum_part(const float *part, int splits, size_t stride, size_t off) {
    // up to 32 independent loads in flight per round; fixed (split-ascending) add order
    float s = 0.f;
    for (int q = 0; q < splits; q += 32) {
        float v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = q + u < splits ? (*(part + (q + u) * stride + off)) : 0.f;
#pragma unroll
        for (int u = 0; u < 32; ++u) s += v[u];
    }
    return s;
}

// sum over the batch of f(b) with 16 samples' loads in flight (fixed add order)
template <class F>
__device__ __forceinline__ float batch_sum(int n, F f) {
    float s = 0.f;
    for (int b0 = 0; b0 < n; b0 += 16) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = b0 + u < n ? f(b0 + u) : 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
    }
    return s;
}

// summed gradient of parameter i (sh: its bf16 shadow index, -1 if none)
__device__ __forceinline__ float grad_of(const OptArgs &a, int64_t i, int64_t &sh) {
    sh = -1;
    if (i < P_B1) {
        int o = (int)(i >> 8), k = (int)(i & 255);
        sh = S_W1 + i;
        const int row = a.w1_perm ? w1_perm(k) : k;  // TMA conv1 wgrad rows are permuted
        return sum_part(a.part1, a.s1, 32 * 257, (size_t)o * 257 + row) * (1.0f / 255.0f);
    }
    if (i < P_W2) return sum_part(a.part1, a.s1, 32 * 257, (size_t)(i - P_B1) * 257 + 256);
    if (i < P_B2) {
        int64_t r = i - P_W2;
        sh = S_W2 + r;
        return sum_part(a.part2, a.s2, 64 * 513, (size_t)(r >> 9) * 513 + (r & 511));
    }
    if (i < P_W3) return sum_part(a.part2, a.s2, 64 * 513, (size_t)(i - P_B2) * 513 + 512);
    if (i < P_B3) {
        int64_t r = i - P_W3;
        sh = S_W3 + r;
        return sum_part(a.part3, a.s3, 64 * 577, (size_t)(r / 576) * 577 + (r % 576));
    }
    if (i < P_W4) return sum_part(a.part3, a.s3, 64 * 577, (size_t)(i - P_B3) * 577 + 576);
    if (i < P_B4) {
        sh = S_W4 + (i - P_W4);
        return (*(a.grad4 + (i - P_W4)));
    }
    const size_t fstride = (size_t)(a.A + 2) * 512;
    if (i < P_W5) {
        const int j = (int)(i - P_B4);
        if (a.fcpart) return sum_part(a.fcpart, a.fcchunks, fstride, (size_t)a.A * 512 + j);
        return batch_sum(a.n, [&](int b) { return (*(a.dh1 + (size_t)b * 512 + j)); });
    }
    if (i < p_b5(a.A)) {
        const int64_t r = i - P_W5;
        const int aa = (int)(r >> 9), j = (int)(r & 511);
        if (a.fcpart) return sum_part(a.fcpart, a.fcchunks, fstride, (size_t)aa * 512 + j);
        return batch_sum(a.n, [&](int b) {
            const float x = (*(a.td + b * 3 + 1)) * (*(a.h1 + (size_t)b * 512 + j));
            return (*(a.act + b)) == aa ? x : 0.f;
        });
    }
    const int aa = (int)(i - p_b5(a.A));
    if (a.fcpart) return sum_part(a.fcpart, a.fcchunks, fstride, (size_t)(a.A + 1) * 512 + aa);
    return batch_sum(a.n, [&](int b) { return (*(a.act + b)) == aa ? (*(a.td + b * 3 + 1)) : 0.f; });
}

constexpr int FC_CHUNK = 16;            // samples per fc2 / fc1-bias gradient partial (qnet.cu)
constexpr int FC_PART_MIN_BATCH = 129;  // batches from which the fc2 / fc1-bias sums use partials

// centered RMSProp, kappa inside the square root (_kernels_numba.py:98-111)
__device__ __forceinline__ void rms(const OptArgs &a, float g, float m, float v, float p,
                                    float &m2, float &v2, float &p2) {
    m2 = a.rho * m + (1.0f - a.rho) * g;
    v2 = a.rho * v + (1.0f - a.rho) * g * g;
    p2 = p - a.lr * g * rsqrtf(v2 - m2 * m2 + a.kappa);
}

// one parameter's update; upd = the update id reported on a non-finite gradient
// a parameter's optimizer state, loaded ahead of the gradient (the one-shot optimizer
// kernels issue these loads before their dependency wait: the previous update wrote them)
struct OptPre {
    float m, v, p;
};
__device__ __forceinline__ OptPre opt_load(const OptArgs &a, int64_t i) {
    return OptPre{(*(a.m + i)), (*(a.v + i)), (*(a.p + i))};
}
__device__ __forceinline__ void opt_finish(const OptArgs &a, int64_t i, int upd, const OptPre &pre, float g,
                                           int64_t sh) {
    const float m = pre.m, v = pre.v, p = pre.p;
    float m2, v2, p2;
    rms(a, g, m, v, p, m2, v2, p2);
    a.m2[i] = m2;
    a.v2[i] = v2;
    a.p2[i] = p2;
    if (sh >= 0) a.shadow[sh] = __float2bfloat16_rn(p2);
    if (i < P_B1) a.shadow[S_W1P + (i >> 8) * 256 + w1_perm((int)(i & 255))] = __float2bfloat16_rn(p2);
    if (a.grad_out) a.grad_out[i] = g;
    if (!isfinite(g)) atomicMin(a.flag, upd);
}
__device__ __forceinline__ void opt_param(const OptArgs &a, int64_t i, int upd, const OptPre &pre) {
    int64_t sh;
    const float g = grad_of(a, i, sh);
    opt_finish(a, i, upd, pre, g, sh);
}
__device__ __forceinline__ void opt_param(const OptArgs &a, int64_t i, int upd) {
    opt_param(a, i, upd, opt_load(a, i));
}

}  // namespace pq
