// Host-side synthetic frame environments + epsilon-greedy selection (the samplers of
// the reference executor, executor.py:237-249 / agent.py:53-66, run on CPU threads in
// the paper's hardware picture).  Used by the end-to-end path: every lockstep block
// the host steps W envs on the Q-rows read back from the GPU and ships the new frames
// to HBM.  Same algorithms as csrc/env.cu and oracle/envs.py, so the two executors
// produce identical trajectories from identical Q-rows.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/paraq_b200.h"

namespace {

typedef unsigned __int128 u128;
const u128 MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

struct Pcg {
    uint64_t *s;  // {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}
    uint64_t next64() {
        u128 st = (((u128)s[0]) << 64) | s[1];
        u128 inc = (((u128)s[2]) << 64) | s[3];
        st = st * MULT + inc;
        s[0] = (uint64_t)(st >> 64);
        s[1] = (uint64_t)st;
        uint64_t x = s[0] ^ s[1];
        unsigned rot = (unsigned)(s[0] >> 58);
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
    uint32_t next32() {
        if (s[4]) {
            s[4] = 0;
            return (uint32_t)s[5];
        }
        uint64_t v = next64();
        s[4] = 1;
        s[5] = v >> 32;
        return (uint32_t)v;
    }
    double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
    uint32_t bounded(uint32_t n) {
        if (n <= 1) return 0;
        uint64_t m = (uint64_t)next32() * n;
        uint32_t left = (uint32_t)m;
        if (left < n) {
            uint32_t threshold = (0u - n) % n;
            while (left < threshold) {
                m = (uint64_t)next32() * n;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline void make_frame(uint64_t key, int64_t episode, int t, int action, uint8_t *dst) {
    uint64_t base = splitmix64(splitmix64(splitmix64(key) ^ (uint64_t)episode) ^
                               (((uint64_t)t << 8) | (uint64_t)action));
    uint64_t *d = reinterpret_cast<uint64_t *>(dst);
    for (int p = 0; p < PQ_FRAME_BYTES / 8; ++p) d[p] = splitmix64(base + (uint64_t)p);
}

inline double epsilon_at(int64_t t, double start, double end, int64_t anneal) {
    if (t >= anneal || anneal == 1) return end;
    double frac = (double)(t - 1) / (double)(anneal - 1);  // built with -ffp-contract=off
    return start + (end - start) * frac;
}

}  // namespace

extern "C" {

/* Reset all W envs (episode start): reset frames go to consecutive frame sequence
 * numbers starting at *seq (advanced); frames_out [W][7056]; stacks [W][4]. */
int pq_henv_reset(pq_henv *e, int W, int64_t *seq, int64_t frame_capacity, uint8_t *frames_out,
                  int32_t *stacks) {
    for (int j = 0; j < W; ++j) {
        e[j].episode += 1;
        e[j].t = 0;
        e[j].ep_return = 0.0;
        int32_t slot = (int32_t)((*seq + j) % frame_capacity);
        make_frame(e[j].key, e[j].episode, 0, 255, frames_out + (size_t)j * PQ_FRAME_BYTES);
        stacks[j * 4 + 0] = stacks[j * 4 + 1] = stacks[j * 4 + 2] = -1;
        stacks[j * 4 + 3] = slot;
    }
    *seq += W;
    return 0;
}

/* One lockstep block for W host envs given their Q rows (q [W][A], fp32):
 * select_action on each env's own stream, env.step, transition record (records
 * [W][8]), episode bookkeeping and reset.  New frames are written to frames_out in
 * order with consecutive sequence numbers from *seq (returned count *nframes);
 * stacks [W][4] are updated in place to the next states. */
int pq_henv_step(pq_henv *e, int W, const float *q, int A, int episode_length, double terminal_p,
                 int64_t t_label0, double eps_start, double eps_end, int64_t eps_anneal,
                 int64_t *seq, int64_t frame_capacity, uint8_t *frames_out, int *nframes,
                 int32_t *stacks, int32_t *records, int64_t *ep_labels, double *ep_rets,
                 int *n_eps) {
    int nf = 0;
    for (int j = 0; j < W; ++j) {
        Pcg g{e[j].pcg};
        const int64_t t_label = t_label0 + j;
        const float *qr = q + (size_t)j * A;
        int act;
        if (g.random() < epsilon_at(t_label, eps_start, eps_end, eps_anneal)) {
            act = (int)g.bounded((uint32_t)A);
        } else {
            act = 0;
            for (int a = 1; a < A; ++a)
                if (qr[a] > qr[act]) act = a;
        }
        const double reward = g.random();
        const bool term = g.random() < terminal_p;
        const int t = e[j].t + 1;
        const int32_t fs = (int32_t)((*seq + nf) % frame_capacity);
        make_frame(e[j].key, e[j].episode, t, act, frames_out + (size_t)nf * PQ_FRAME_BYTES);
        ++nf;
        const bool trunc = !term && t >= episode_length;
        int32_t *rec = records + (size_t)j * PQ_REC_INTS;
        int32_t *st = stacks + j * 4;
        uint64_t rbits;
        memcpy(&rbits, &reward, 8);
        rec[0] = st[0], rec[1] = st[1], rec[2] = st[2], rec[3] = st[3], rec[4] = fs;
        rec[5] = act | (term ? 1 << 16 : 0);  // action | bootstrap terminal << 16
        rec[6] = (int32_t)(uint32_t)rbits, rec[7] = (int32_t)(uint32_t)(rbits >> 32);  // f64 reward
        e[j].ep_return += reward;
        if (term || trunc) {
            ep_labels[*n_eps] = t_label;
            ep_rets[*n_eps] = e[j].ep_return;
            *n_eps += 1;
            e[j].ep_return = 0.0;
            e[j].episode += 1;
            e[j].t = 0;
            const int32_t rs = (int32_t)((*seq + nf) % frame_capacity);
            make_frame(e[j].key, e[j].episode, 0, 255, frames_out + (size_t)nf * PQ_FRAME_BYTES);
            ++nf;
            st[0] = st[1] = st[2] = -1;
            st[3] = rs;
        } else {
            e[j].t = t;
            st[0] = st[1], st[1] = st[2], st[2] = st[3], st[3] = fs;
        }
    }
    *seq += nf;
    *nframes = nf;
    return 0;
}

}  // extern "C"
