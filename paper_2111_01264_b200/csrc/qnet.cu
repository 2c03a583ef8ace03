// Nature-CNN Q-network forward, DQN learner step and fused centered RMSProp.
//
// Reference path restated (pkg/src/paraq):
//   forward          nn.py:123-131   -> F1..F4 implicit GEMMs (tcgen05) + k_head
//   td_targets       agent.py:69-81  -> k_head (target forward max, bootstrap)
//   gradient         nn.py:134-170   -> k_head (output_delta, fc2 back-prop) +
//                                       B4w/B4d, B3w/B3d, B2w/B2d, B1w GEMMs
//   x n rescale      agent.py:103-104 -> delta = q - target (summed-gradient convention)
//   rmsprop_step     nn.py:173-203   -> k_optimizer (split-K reduction + RMSProp + bf16
//                                       shadow refresh + non-finite flag)
#include <climits>
#include <cstdio>
#include <cstring>

#include "../../include/paraq_b200.h"
#include "gemm.cuh"
#include "learn_parts.cuh"
#include "qnet.cuh"

namespace pq {



thread_local char g_err[512] = "";
int set_err(const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return 1;
}
int cuda_err(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return 0;
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return 2;
}
#define PQ_CHECK(expr, where)                          \
    do {                                               \
        int _rc = cuda_err((expr), where);             \
        if (_rc) return _rc;                           \
    } while (0)

// TMA-engine GEMMs (learner.cu); PQ_TMA=0 selects the cp.async engine for every GEMM
int tma_conv3_fwd(const pq_net *nets, bf16 *const *act2, bf16 *const *act3, int groups, int n, cudaStream_t st);
int tma_fc1_fwd(const pq_net *nets, bf16 *const *act3, float *const *part, int splits, int groups, int n,
                cudaStream_t st);
int tma_fc1_fwd_acc7(const pq_net *nets, bf16 *const *act3, float *const *part, int groups, int n, cudaStream_t st);
int tma_fc1_fwd_resident(const pq_net *nets, bf16 *const *act3, float *const *part, int splits, int groups, int n,
                         cudaStream_t st);
int tma_fc1_dgrad_resident(const pq_net &th, const bf16 *dh1_bf, const bf16 *act3, bf16 *dY3, int n,
                           cudaStream_t st, bf16 *dY3p);
int tma_conv3_dgrad_shift(const pq_net &th, const bf16 *dY3p, const bf16 *act2, bf16 *dY2, bf16 *dY2p, bf16 *dY2q,
                          int n, cudaStream_t st);
int tma_fc1_dgrad(const pq_net &th, const bf16 *dh1_bf, const bf16 *act3, bf16 *dY3, int n, cudaStream_t st);
int tma_conv3_dgrad(const pq_net &th, const bf16 *dY3, const bf16 *act2, bf16 *dY2, int n, cudaStream_t st,
                    bf16 *dY2p, bf16 *dY2q);
int tma_conv2_wgrad_shift(const bf16 *act1s2, const bf16 *dY2q, float *part2, int kc, int splits, int n,
                          cudaStream_t st);
int tma_conv2_dgrad_shift(const pq_net &th, const bf16 *dY2p, const bf16 *act1, bf16 *dY1, int n, int pad21,
                          cudaStream_t st, int mask_s2);
int tma_conv3_wgrad(const bf16 *act2, const bf16 *dY3, float *part3, int kc, int splits, int n, cudaStream_t st);
int tma_conv2_dgrad(const pq_net &th, const bf16 *dY2, const bf16 *act1, bf16 *dY1, int n, cudaStream_t st,
                    int pad21);
int tma_frames_s2d(const uint8_t *ring, const int32_t *refs, const int64_t *map, const int32_t *counter,
                   int map_stride, int ref_stride, int ref_off, int nframes, int n, bf16 *out, cudaStream_t st);
int tma_conv1_fwd(const pq_net *nets, const bf16 *s2d, int nframes, const int *c0, bf16 *const *act1, int groups,
                  int n, cudaStream_t st);
int tma_conv1_shift(const pq_net *nets, const bf16 *s2d, int nframes, const int *c0, bf16 *const *act1,
                    int groups, int n, int a_early, int w_early, cudaStream_t st, bf16 *const *act1s2);
int tma_conv2_shift(const pq_net *nets, bf16 *const *act1s2, bf16 *const *act2, int groups, int n, cudaStream_t st);
int tma_conv3_shift(const pq_net *nets, bf16 *const *act2, bf16 *const *act3, int groups, int n, cudaStream_t st);
int tma_conv1_wgrad(const bf16 *s2d, int nframes, const bf16 *dY1, float *part1, int kc, int splits, int n,
                    cudaStream_t st);
int tma_conv1_wgrad_shift(const bf16 *s2d, int nframes, const bf16 *dY1p, float *part1, int kc, int splits,
                          int n, cudaStream_t st);
// conv1 forward / weight gradient by row-shifted UMMA descriptors over the s2d stacks
// (PQ_C1SHIFT=0: the im2col TMA kernels)
static bool conv1_shift() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("PQ_C1SHIFT");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}
// Engine per GEMM (measured, profiles/r1_engine_compare.md): below batch 128 every CTA
// owns ~one tile and the cp.async engine's shorter first-load latency wins inside the
// CUDA graph; from 128 up the warp-specialised TMA engine overlaps tiles and wins.
// PQ_TMA=0 / 1 forces one engine.
static bool use_tma(int n) {
    static int mode = -2;
    if (mode == -2) {
        const char *e = getenv("PQ_TMA");
        mode = e ? (e[0] == '0' ? 0 : 1) : -1;
    }
    return mode >= 0 ? mode == 1 : n >= 128;
}

// fc1 forward with the split sums reduced in TMEM (learner.cu k_fc1_acc7: one CTA per
// (network, 128-unit tile, 64 samples)) once that is at least 128 CTAs -- the learner's two
// networks from batch 512, the acting forward (one network) from 1024; below, the
// resident-A split-K kernel has the parallelism (PQ_F7=0: always it).  The head / acting
// kernels then read 1 split.
static bool fc1_acc7(int n, int groups) {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("PQ_F7");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1 && groups * 4 * ((n + 63) / 64) >= 128 && use_tma(n) && conv1_shift();
}
int fc1_splits(int n, int groups) { return fc1_acc7(n, groups) ? 1 : FC1_SPLITS; }

// ------------------------------------------------------------------ workspace
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct WS {
    bf16 *act1[2], *act2[2], *act3[2];
    float *fc1part[2];
    float *q, *h1, *dh1, *td;
    bf16 *dh1_bf, *dh1T;
    int32_t *act;
    bf16 *dY3, *dY2, *dY1;
    bf16 *dY1p;  // conv2's data gradient on the padded 21 x 21 grid (TMA engine; pad rows stay 0)
    bf16 *dY2p;  // conv3's data gradient on the padded 11 x 11 grid (TMA engine; pad rows stay 0)
    bf16 *act1s2[2];  // act1 as 2x2 space-to-depth [n][10][10][128] (TMA engine, shifted conv2)
    bf16 *dY2q;       // conv3's data gradient on the 10 x 10 grid (zero rows at 9; shifted conv2 wgrad)
    bf16 *dY3p;       // fc1's data gradient on the zero-padded 11 x 11 grid (shifted conv3 dgrad)
    float *part1, *part2, *part3, *grad4;
    uint32_t *done;  // [3] CTA completion counters (unused, acting, head)
    int64_t *idx_cur;  // the step's sampled slots (stashed by the head)
    int32_t *upd_cur;  // the step's update id (stashed by the head)
    int32_t *step_stash;  // the step's update id, copied by the step's first launch (read
                          // before the dependency wait by later launches of the step)
    float *fcpart;     // fc2 / fc1-bias gradient partials per 64-sample chunk (large batches)
    bf16 *s2d;         // space-to-depth frame stacks [n][21][21][80] (TMA conv1, large batches)
    int n8;
    size_t bytes;
};

static WS carve(void *base, int N, int A) {
    WS w;
    size_t off = 0;
    char *b = static_cast<char *>(base);
    auto take = [&](size_t bytes) -> void * {
        void *p = b ? b + off : nullptr;
        off += al(bytes);
        return p;
    };
    int n8 = (N + 7) & ~7;
    w.n8 = n8;
    for (int g = 0; g < 2; ++g) {
        w.act1[g] = (bf16 *)take((size_t)N * 400 * 32 * 2);
        w.act2[g] = (bf16 *)take((size_t)N * 81 * 64 * 2);
        w.act3[g] = (bf16 *)take((size_t)N * 3136 * 2);
        w.fc1part[g] = (float *)take((size_t)FC1_SPLITS * N * 512 * 4);
    }
    w.q = (float *)take((size_t)2 * N * A * 4);
    w.h1 = (float *)take((size_t)N * 512 * 4);
    w.dh1 = (float *)take((size_t)N * 512 * 4);
    w.td = (float *)take((size_t)N * 3 * 4);
    w.dh1_bf = (bf16 *)take((size_t)N * 512 * 2);
    w.dh1T = (bf16 *)take((size_t)512 * n8 * 2);
    w.act = (int32_t *)take((size_t)N * 4);
    w.dY3 = (bf16 *)take((size_t)N * 3136 * 2);
    w.dY2 = (bf16 *)take((size_t)N * 81 * 64 * 2);
    w.dY1 = (bf16 *)take((size_t)N * 400 * 32 * 2);
    w.part1 = (float *)take((size_t)P1_MAX_SPLITS * 32 * 257 * 4);
    w.part2 = (float *)take((size_t)MAX_SPLITS * 64 * 513 * 4);
    w.part3 = (float *)take((size_t)MAX_SPLITS * 64 * 577 * 4);
    w.grad4 = (float *)take((size_t)512 * 3136 * 4);
    w.done = (uint32_t *)take(3 * sizeof(uint32_t));
    w.idx_cur = (int64_t *)take((size_t)N * 8);
    w.upd_cur = (int32_t *)take(sizeof(int32_t));
    w.step_stash = (int32_t *)take(sizeof(int32_t));
    w.fcpart = (float *)take((size_t)((N + FC_CHUNK - 1) / FC_CHUNK) * (A + 2) * 512 * 4);
    w.s2d = N >= 128 ? (bf16 *)take((size_t)N * 441 * 80 * 2) : nullptr;
    w.dY1p = N >= 128 ? (bf16 *)take((size_t)N * 441 * 32 * 2) : nullptr;  // zeroed with the workspace
    w.dY2p = N >= 128 ? (bf16 *)take((size_t)N * 121 * 64 * 2) : nullptr;
    for (int g = 0; g < 2; ++g) w.act1s2[g] = N >= 128 ? (bf16 *)take((size_t)N * 100 * 128 * 2) : nullptr;
    w.dY2q = N >= 128 ? (bf16 *)take((size_t)N * 100 * 64 * 2) : nullptr;
    w.dY3p = (bf16 *)take((size_t)N * 121 * 64 * 2);  // also the batch-32 shifted conv3 dgrad (Dg3ShiftOp)
    w.bytes = off;
    return w;
}

// ------------------------------------------------------------------ forward GEMMs
struct FwdInput {  // frame-stack addressing of one group
    const uint8_t *ring;
    const int32_t *refs;
    const int64_t *map;
    const int32_t *counter;  // optional: map += *counter * map_stride
    int map_stride;
    int ref_stride, ref_off;
};


static LoadFrames frames_loader(const FwdInput &in, int n) {
    return frames(in.ring, in.refs, in.map, in.counter, in.map_stride, n, in.ref_stride, in.ref_off);
}

static int choose_bn(int n) {
    return n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256;
}

template <class LA, class LB, class EP, bool AMN, bool BMN, int PF = 0>
static cudaError_t launch_bn(int bn, const GemmArgs<LA, LB, EP> &g, int groups, cudaStream_t st) {
    switch (bn) {
        case 16: return launch_gemm<16, AMN, BMN, 0, PF>(g, groups, st);
        case 32: return launch_gemm<32, AMN, BMN, 0, PF>(g, groups, st);
        case 64: return launch_gemm<64, AMN, BMN, 0, PF>(g, groups, st);
        case 128: return launch_gemm<128, AMN, BMN, 0, PF>(g, groups, st);
        default: return launch_gemm<256, AMN, BMN, 0, PF>(g, groups, st);
    }
}

// F1..F4 for `groups` parameter sets (group 0 / 1 = online / target in the learner)
// early_frames: the learner -- its frames / records are never written by the kernel
// before it (only the acting kernel writes frames, and it triggers its dependents
// early), so conv1 builds its frame table and requests frames before the wait
static int forward_gemms(const pq_net *nets, const FwdInput *ins, int groups, int n, const WS &w,
                         cudaStream_t st, bool early_frames = false) {
    if (use_tma(n) && w.s2d) {  // F1 on the TMA engine over the space-to-depth stacks
        // learner: frames f0..f4 once, online = channels 0..63, target = 16..79
        const int nframes = groups == 2 ? 5 : 4;
        const int c0[2] = {0, 16};
        bf16 *a1[2] = {w.act1[0], w.act1[1]};
        if (int rc = tma_frames_s2d(ins[0].ring, ins[0].refs, ins[0].map, ins[0].counter, ins[0].map_stride,
                                    ins[0].ref_stride, ins[0].ref_off, nframes, n, w.s2d, st))
            return rc;
        if (conv1_shift()) {  // the s2d kernel just wrote the frames; weights are two launches back
            if (int rc = tma_conv1_shift(nets, w.s2d, nframes, c0, a1, groups, n, 0, 1, st, w.act1s2)) return rc;
        } else if (int rc = tma_conv1_fwd(nets, w.s2d, nframes, c0, a1, groups, n, st)) {
            return rc;
        }
    } else {  // F1: conv1 8x8/4 over uint8 frames (K = 256), bias + ReLU, x 1/255
        GemmArgs<LoadFrames, LoadDense, EpiBiasRelu> g{};
        for (int q = 0; q < groups; ++q) {
            g.a[q] = frames_loader(ins[q], n);
            g.b[q] = LoadDense{(const bf16 *)nets[q].shadow + S_W1P, 32, 256, 256};  // permuted K
            g.e[q] = EpiBiasRelu{w.act1[q], nets[q].master + P_B1, n * 400, 32, 32, 1.0f / 255.0f};
        }
        g.M = n * 400, g.N = 32, g.K = 256, g.kc_per_split = 4, g.splits = 1, g.ones_at = -1;
        if (early_frames)
            PQ_CHECK((launch_gemm<32, false, false, 3, 1>(g, groups, st)), "conv1 forward");
        else
            PQ_CHECK((launch_gemm<32, false, false, 3>(g, groups, st)), "conv1 forward");
    }
    bf16 *a2[2] = {w.act2[0], w.act2[1]}, *a3[2] = {w.act3[0], w.act3[1]};
    float *pt[2] = {w.fc1part[0], w.fc1part[1]};
    if (use_tma(n) && w.s2d && conv1_shift() && w.act1s2[0]) {  // F2 over act1's 2x2 space-to-depth
        bf16 *s2[2] = {w.act1s2[0], w.act1s2[1]};
        if (int rc = tma_conv2_shift(nets, s2, a2, groups, n, st)) return rc;
    } else {  // F2: conv2 4x4/2 over 20x20x32 (K = 512)
        GemmArgs<LoadIm2col, LoadDense, EpiBiasRelu> g{};
        for (int q = 0; q < groups; ++q) {
            g.a[q] = im2col(w.act1[q], n, 20, 20, 32, 4, 2, 9, 9);
            g.b[q] = LoadDense{(const bf16 *)nets[q].shadow + S_W2, 64, 512, 512};
            g.e[q] = EpiBiasRelu{w.act2[q], nets[q].master + P_B2, n * 81, 64, 64, 1.0f};
        }
        g.M = n * 81, g.N = 64, g.K = 512, g.kc_per_split = 8, g.splits = 1, g.ones_at = -1;
        PQ_CHECK((launch_gemm<64, false, false, 0, 2>(g, groups, st)), "conv2 forward");
    }
    // engine per GEMM (measured, profiles/r1_engine_compare.md): the TMA im2col conv3
    // forward wins once a CTA has several tiles; at small batch the cp.async one does
    if (use_tma(n) && conv1_shift()) {  // the 7 x 7 outputs on act2's own 9 x 9 grid
        if (int rc = tma_conv3_shift(nets, a2, a3, groups, n, st)) return rc;
    } else if (use_tma(n)) {
        if (int rc = tma_conv3_fwd(nets, a2, a3, groups, n, st)) return rc;
    } else {  // F3: conv3 3x3/1 over 9x9x64 (K = 576)
        GemmArgs<LoadIm2col, LoadDense, EpiBiasRelu> g{};
        for (int q = 0; q < groups; ++q) {
            g.a[q] = im2col(w.act2[q], n, 9, 9, 64, 3, 1, 7, 7);
            g.b[q] = LoadDense{(const bf16 *)nets[q].shadow + S_W3, 64, 576, 576};
            g.e[q] = EpiBiasRelu{w.act3[q], nets[q].master + P_B3, n * 49, 64, 64, 1.0f};
        }
        g.M = n * 49, g.N = 64, g.K = 576, g.kc_per_split = 9, g.splits = 1, g.ones_at = -1;
        PQ_CHECK((launch_gemm<64, false, false, 0, 2>(g, groups, st)), "conv3 forward");
    }
    if (fc1_acc7(n, groups)) return tma_fc1_fwd_acc7(nets, a3, pt, groups, n, st);
    if (use_tma(n) && conv1_shift())  // W4 chunks resident per CTA
        return tma_fc1_fwd_resident(nets, a3, pt, FC1_SPLITS, groups, n, st);
    if (use_tma(n)) return tma_fc1_fwd(nets, a3, pt, FC1_SPLITS, groups, n, st);
    {  // F4: fc1, swapped (D[j][b] = W4[j] . x[b]) with split-K partials [s][b][j]
        GemmArgs<LoadDense, LoadDense, EpiF32T> g{};
        for (int q = 0; q < groups; ++q) {
            g.a[q] = LoadDense{(const bf16 *)nets[q].shadow + S_W4, 512, 3136, 3136};
            g.b[q] = LoadDense{w.act3[q], n, 3136, 3136};
            g.e[q] = EpiF32T{w.fc1part[q], 512, n, 512, (size_t)n * 512};
        }
        g.M = 512, g.N = n, g.K = 3136, g.kc_per_split = 49 / FC1_SPLITS, g.splits = FC1_SPLITS,
        g.ones_at = -1;
        PQ_CHECK((launch_bn<LoadDense, LoadDense, EpiF32T, false, false, 1>(choose_bn(n), g, groups, st)),
                 "fc1 forward");
    }
    return 0;
}

// ------------------------------------------------------------------ head kernel
// one 256-thread CTA per sample (learn_parts.cuh: head_sample)
// last CTA of a grid bumps a device step counter (replaces a separate launch)
__device__ __forceinline__ void last_block_bump(int32_t *counter, uint32_t *done) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        *counter += 1;
        *done = 0;
        __threadfence();
    }
}

// The learner's head also stashes the step's sampled slots and update id, then advances
// the step counter (last CTA): later kernels of the step read the stash, so the
// optimizer can be split across streams without racing on the counter.
__global__ void __launch_bounds__(HEAD_THREADS) k_head(const HeadArgs a, int32_t *bump, uint32_t *done) {
    TlProbe tp;
    ct_begin();
    auto wait = [&] {
        griddep_wait();
        griddep_launch();
        tp.waited();
        ct_mark(1);
    };
    head_sample<FC1_SPLITS>(a, blockIdx.x, wait);  // (1 split: k_head_block)
    if (bump) last_block_bump(bump, done);
    tp.done('H');
    ct_end('H');
}

// large batches (fc1 sums reduced by the forward GEMM, k_fc1_acc7): HEAD_BLOCK samples per
// CTA (learn_parts.cuh: head_block); a kernel of its own so the batch-32 head stays lean
__global__ void __launch_bounds__(HEAD_THREADS) k_head_block(const HeadArgs a, int32_t *bump, uint32_t *done) {
    TlProbe tp;
    head_block<1, HEAD_BLOCK>(a, blockIdx.x * HEAD_BLOCK, [&] {
        griddep_wait();
        griddep_launch();
        tp.waited();
    });
    if (bump) last_block_bump(bump, done);
    tp.done('H');
}

// batches from 512 whose fc1 sums are still split-K partials (below k_fc1_acc7's range):
// the same HEAD_BLOCK samples per CTA, reducing the FC1_SPLITS partials per sample like
// k_head (fc2 weights read once per HEAD_BLOCK samples instead of once per sample)
constexpr int HEAD_BLOCK_SPLIT_MIN = 512;  // measured: slower at 128 / 256 (fewer CTAs)
__global__ void __launch_bounds__(HEAD_THREADS) k_head_block_split(const HeadArgs a, int32_t *bump, uint32_t *done) {
    TlProbe tp;
    head_block<FC1_SPLITS, HEAD_BLOCK>(a, blockIdx.x * HEAD_BLOCK, [&] {
        griddep_wait();
        griddep_launch();
        tp.waited();
    });
    if (bump) last_block_bump(bump, done);
    tp.done('H');
}

static bool fused_backward(int n, const pq_learn_args *la, float *grad_only);

// bump_here: the step counter advances in the head (split or fused optimizer schedules);
// otherwise at the tail of the one optimizer launch
static int head(const pq_net *nets, int groups, int n, int A, const WS &w, int learner,
                const pq_learn_args *la, cudaStream_t st, bool bump_here = false) {
    HeadArgs h{};
    for (int g = 0; g < groups; ++g) {
        h.part[g] = w.fc1part[g];
        h.master[g] = nets[g].master;
    }
    h.groups = groups, h.n = n, h.A = A, h.n8 = w.n8, h.splits = fc1_splits(n, groups);
    h.block = h.splits == 1 ? HEAD_BLOCK : 1;
    h.learner = learner;
    h.q_out = w.q, h.h1 = w.h1, h.dh1 = w.dh1, h.td = w.td, h.dh1_bf = w.dh1_bf, h.dh1T = w.dh1T;
    h.act_out = w.act;
    if (la) {
        h.records = la->records, h.idx = la->idx, h.idx_base = la->idx_base;
        h.counter = la->update_counter, h.ext_targets = la->ext_targets;
        h.ext_actions = la->ext_actions, h.gamma = la->gamma, h.huber = la->huber;
        h.q_copy = la->q_out, h.td_copy = la->td_out;
        h.idx_cur = w.idx_cur, h.upd_cur = w.upd_cur;
    }
    int32_t *bump = (la && learner && !la->idx && la->update_counter && bump_here) ? la->update_counter : nullptr;
    if (h.block == HEAD_BLOCK)
        return cuda_err(launch_k(k_head_block, dim3((n + HEAD_BLOCK - 1) / HEAD_BLOCK), dim3(HEAD_THREADS), 0, st, h,
                                 bump, w.done + 2),
                        "head");
    if (h.splits == FC1_SPLITS && n >= HEAD_BLOCK_SPLIT_MIN)
        return cuda_err(launch_k(k_head_block_split, dim3((n + HEAD_BLOCK - 1) / HEAD_BLOCK), dim3(HEAD_THREADS), 0,
                                 st, h, bump, w.done + 2),
                        "head");
    return cuda_err(launch_k(k_head, dim3(n), dim3(HEAD_THREADS), 0, st, h, bump, w.done + 2), "head");
}

// fc2 / fc1-bias gradient partials of one 64-sample chunk (blockIdx.x), 512 threads =
// hidden units j: rows 0..A-1 = sum_b [a_b = a] delta_b h1[b][j] (fc2 weights), row A =
// sum_b dh1[b][j] (fc1 bias), row A+1 = sum_b [a_b = a] delta_b (fc2 bias, columns a < A).
// Fixed order within and across chunks (deterministic); large batches only.
__global__ void __launch_bounds__(512) k_fc2_partials(const float *h1, const float *dh1, const float *td,
                                                      const int32_t *act, int n, int A, float *part) {
    TlProbe tp;
    griddep_wait();
    griddep_launch();
    tp.waited();
    __shared__ float s_d[FC_CHUNK];
    __shared__ int s_a[FC_CHUNK];
    // per-action sums in shared memory, column j owned by thread j (conflict-free): one
    // add per sample instead of a predicated add for every action
    extern __shared__ float s_acc_raw[];  // [A][512] (dynamic: up to 64 KB)
    float(*s_acc)[512] = reinterpret_cast<float(*)[512]>(s_acc_raw);
    const int b0 = blockIdx.x * FC_CHUNK, nb = min(FC_CHUNK, n - b0), j = threadIdx.x;
    if (j < nb) {
        s_d[j] = td[(b0 + j) * 3 + 1];
        s_a[j] = act[b0 + j];
    }
    for (int aa = 0; aa < A; ++aa) s_acc[aa][j] = 0.f;
    __syncthreads();
    float ab = 0.f, bb = 0.f;
    // 16 samples' loads in flight per round (a one-sample loop is load-latency bound);
    // the adds stay in sample order
    constexpr int U = 16;
    for (int q = 0; q < nb; q += U) {
        float hv[U], dv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = q + u < nb;
            hv[u] = ok ? h1[(size_t)(b0 + q + u) * 512 + j] : 0.f;
            dv[u] = ok ? dh1[(size_t)(b0 + q + u) * 512 + j] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (q + u >= nb) break;
            const int b = q + u;
            const int ab_ = s_a[b];
            s_acc[ab_][j] += s_d[b] * hv[u];
            ab += dv[u];
            if (j < A && ab_ == j) bb += s_d[b];
        }
    }
    float *out = part + (size_t)blockIdx.x * (A + 2) * 512;
    for (int aa = 0; aa < A; ++aa) out[aa * 512 + j] = s_acc[aa][j];
    out[A * 512 + j] = ab;
    if (j < A) out[(A + 1) * 512 + j] = bb;
    tp.done('P');
}

// ------------------------------------------------------------------ optimizer

// the parameters in [lo1, hi1) and [lo2, hi2), one per thread (learn_parts.cuh: opt_param)
// The single-stream learner's update launch: blocks [0, nb1) update conv1 (one parameter
// per thread) once the conv1 weight gradient -- the launch before -- is complete; the
// other blocks update conv2 / conv3 / fc1-bias / fc2 (pt parameters per thread, strided)
// without waiting: their gradients were complete two or more launches back and their last
// readers (the conv2 / conv3 data gradients) likewise, so they run while conv1's weight
// gradient drains (on the SMs it leaves free) and as its CTAs exit.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_opt_tail(const OptArgs a, int nb1, int pt, int first1) {
    ct_begin();
    const int upd = a.counter ? *a.counter : 0;
    const int nb2 = (int)gridDim.x - nb1;
    // first1: the no-wait blocks take the low block ids (scheduled first, onto the SMs the
    // conv1 weight gradient leaves free); else the conv1 blocks do
    const int bid = first1 ? ((int)blockIdx.x < nb2 ? (int)blockIdx.x + nb1 : (int)blockIdx.x - nb2) : (int)blockIdx.x;
    if (bid < nb1) {
        const int64_t i = P_W1 + (int64_t)bid * 256 + threadIdx.x;
        const bool live = i < P_W2;
        const OptPre pre = live ? opt_load(a, i) : OptPre{};
        griddep_wait();
        griddep_launch();
        ct_mark(1);
        if (live) {
            int64_t sh;
            const float g = grad_of(a, i, sh);
            ct_mark(2);
            opt_finish(a, i, upd, pre, g, sh);
        }
        ct_end('T', 0);
        return;
    }
    griddep_launch();
    ct_mark(1);
    const int64_t n2a = P_W4 - P_W2, n2 = n2a + (a.total - P_B4);
    const int64_t T = (int64_t)nb2 * 256, t = (int64_t)(bid - nb1) * 256 + threadIdx.x;
    for (int k = 0; k < pt; ++k) {
        const int64_t r0 = t + k * T, nfc = n2 - n2a;
        // first1 == 2: the fc1-bias / fc2 parameters (batch sums at small batches: the
        // slowest) on the first threads
        const int64_t r = first1 == 2 ? (r0 < nfc ? n2a + r0 : r0 - nfc) : r0;
        if (r0 < n2) opt_param(a, r < n2a ? P_W2 + r : P_B4 + (r - n2a), upd);
    }
    ct_end('T', 1);
}

__global__ void __launch_bounds__(256) k_optimizer(const OptArgs a) {
    TlProbe tp;
    ct_begin();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n1 = a.hi1 - a.lo1;
    const int64_t i = t < n1 ? a.lo1 + t : a.lo2 + (t - n1);
    const bool live = t < n1 || i < a.hi2;
    // optimizer state and update id before the wait (written two or more launches back)
    const OptPre pre = live ? opt_load(a, i) : OptPre{};
    const int upd = a.counter ? *a.counter : 0;
    griddep_wait();
    griddep_launch();
    tp.waited();
    ct_mark(1);
    if (live) opt_param(a, i, upd, pre);
    if (a.bump) last_block_bump(a.bump, a.bump_done);
    tp.done('O');
    ct_end('O');
}

// summed gradient of every parameter except fc1's weight (written by the fc1 wgrad GEMM)
__global__ void __launch_bounds__(256) k_grad_only(const OptArgs a) {
    griddep_wait();
    griddep_launch();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = t < P_W4 ? t : P_B4 + (t - P_W4);
    if (i < a.total) {
        int64_t sh;
        a.grad_out[i] = grad_of(a, i, sh);
    }
}

// centered RMSProp of every parameter from a gradient vector, bf16 shadow refresh,
// non-finite flag (rmsprop_step, nn.py:173-203; _kernels_numba.py:98-111)
__global__ void __launch_bounds__(256) k_rmsprop_apply(float *p, float *m, float *v, bf16 *shadow,
                                                       const float *g, int64_t total, float lr, float rho,
                                                       float kappa, int32_t *flag, int upd) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const float gi = g[i];
    const float mi = rho * m[i] + (1.0f - rho) * gi;
    const float vi = rho * v[i] + (1.0f - rho) * gi * gi;
    const float pi = p[i] - lr * gi * rsqrtf(vi - mi * mi + kappa);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
    int64_t sh = -1;
    if (i < P_B1) sh = S_W1 + i;
    else if (i >= P_W2 && i < P_B2) sh = S_W2 + (i - P_W2);
    else if (i >= P_W3 && i < P_B3) sh = S_W3 + (i - P_W3);
    else if (i >= P_W4 && i < P_B4) sh = S_W4 + (i - P_W4);
    if (sh >= 0) shadow[sh] = __float2bfloat16_rn(pi);
    if (i < P_B1) shadow[S_W1P + (i >> 8) * 256 + w1_perm((int)(i & 255))] = __float2bfloat16_rn(pi);
    if (!isfinite(gi) && flag) atomicMin(flag, upd);
}

static int choose_kc(int nchunks, int mtiles, int *splits, int kc_max = 1 << 30) {
    int kc = (nchunks * mtiles + 147) / 148;
    if (kc < 2) kc = 2;
    int need = (nchunks + MAX_SPLITS - 1) / MAX_SPLITS;
    if (kc < need) kc = need;
    // no partial second wave: splits x M tiles jobs within one CTA per SM (the ceiling
    // division above can overshoot by a few jobs, e.g. 150 on 148 SMs at batch 1024)
    while (kc < kc_max && ((nchunks + kc - 1) / kc) * mtiles > 148 && ((nchunks + kc - 1) / kc) * mtiles < 2 * 148) ++kc;
    if (kc > kc_max) kc = kc_max;
    *splits = (nchunks + kc - 1) / kc;
    return kc;
}

// side stream + events for the weight-gradient branch (fork after each data
// gradient, join before the optimizer); also captured into CUDA graphs as branches
struct Fork {
    cudaStream_t side = nullptr, side2 = nullptr;
    cudaEvent_t ev[6] = {};
};
static Fork g_fork[16];

static int get_fork(Fork **out) {
    int dev = 0;
    PQ_CHECK(cudaGetDevice(&dev), "get device");
    Fork &f = g_fork[dev & 15];
    if (!f.side) {  // the weight-gradient branch at the highest stream priority (PQ_SIDE_PRIO=0:
        // default priority): its kernels otherwise wait for SMs behind the main stream's
        // persistent grids and end up on the critical path (batch 1024: 427 -> 405 us/step)
        int lo = 0, hi = 0;
        PQ_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
        const char *e = getenv("PQ_SIDE_PRIO");
        const int prio = (e && e[0] == '0') ? lo : hi;
        PQ_CHECK(cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, prio), "side stream");
        PQ_CHECK(cudaStreamCreateWithPriority(&f.side2, cudaStreamNonBlocking, prio), "side stream 2");
        for (auto &e : f.ev) PQ_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    *out = &f;
    return 0;
}

// grad_only != NULL: write the summed gradient of every parameter there instead of
// updating theta / opt (the data-parallel learner all-reduces it, then pq_rmsprop_apply)
// ---- the backward GEMMs of the cp.async engine (also the fused single-stream schedule)
using B3wOp = GemmOp<64, true, true, 0, 0, LoadIm2col, LoadDense, EpiF32T>;
using B3dOp = GemmOp<64, false, true, 0, 2, LoadTConv, LoadWeightT, EpiMask>;
// fc1 weight gradient + RMSProp, started without waiting for the fc1 data gradient (EpiRms4Late)
using B4wLateOp = GemmOp<64, false, true, 4, 0, LoadDense, LoadDense, EpiRms4Late, TriggerHook>;
using B2wOp = GemmOp<64, true, true, 0, 0, LoadIm2col, LoadDense, EpiF32T>;
using B2dOp = GemmOp<64, false, true, 0, 2, LoadTConvP, LoadWeightTP, EpiMaskP>;
using B1wOp = GemmOp<64, true, true, 3, 1, LoadFrames, LoadDense, EpiF32T>;  // frames before the wait

// B4w + RMSProp: dW4[j][k] = sum_b dh1[b][j] x3[b][k] (contraction over the batch),
// centered RMSProp applied in the epilogue (no fp32 gradient round trip)
template <class EP>
static GemmArgs<LoadDense, LoadDense, EP> args_b4w_rms(const pq_learn_args *la, int n, const WS &w) {
    const pq_net &th = la->theta;
    GemmArgs<LoadDense, LoadDense, EP> g{};
    g.a[0] = LoadDense{w.dh1T, 512, n, w.n8};
    g.b[0] = LoadDense{w.act3[0], n, 3136, 3136};
    EP e{};
    e.p = th.master, e.m = la->opt.m, e.v = la->opt.v;
    e.p2 = la->theta_out.master, e.m2 = la->opt_out.m, e.v2 = la->opt_out.v;
    e.shadow = (bf16 *)la->theta_out.shadow;
    e.grad_out = la->grad_out, e.flag = la->nonfinite, e.counter = w.upd_cur;
    e.lr = la->lr, e.rho = la->rho, e.kappa = la->kappa;
    e.M = 512, e.N = 3136, e.pbase = P_W4, e.sbase = S_W4;
    g.e[0] = e;
    g.M = 512, g.N = 3136, g.K = n, g.kc_per_split = (n + 63) / 64, g.splits = 1, g.ones_at = -1;
    return g;
}
// B3w: dW3^T[k][o] = sum_m P3[m][k] dY3[m][o]; row 576 = ones -> bias grad
static B3wOp::Args args_b3w(const WS &w, int n, int *s3) {
    B3wOp::Args g{};
    g.a[0] = im2col(w.act2[0], n, 9, 9, 64, 3, 1, 7, 7);
    g.b[0] = LoadDense{w.dY3, n * 49, 64, 64};
    g.e[0] = EpiF32T{w.part3, 577, 64, 577, (size_t)64 * 577};
    const int nch = (n * 49 + 63) / 64;
    g.kc_per_split = choose_kc(nch, 5, s3);
    g.M = 577, g.N = 64, g.K = n * 49, g.splits = *s3, g.ones_at = 576, g.ones_extent = n * 49;
    return g;
}
// B3d: dY2 = relu'(x2) * transposed conv3(dY3)
static B3dOp::Args args_b3d(const bf16 *sh, const WS &w, int n) {
    B3dOp::Args g{};
    g.a[0] = tconv(w.dY3, n, 9, 9, 7, 7, 64, 3);
    g.b[0] = weight_t(sh + S_W3, 64, 3, 64);
    g.e[0] = EpiMask{w.dY2, w.act2[0], n * 81, 64, 64};
    g.M = n * 81, g.N = 64, g.K = 576, g.kc_per_split = 9, g.splits = 1, g.ones_at = -1;
    return g;
}
// B2w: dW2^T[k][o] = sum_m P2[m][k] dY2[m][o]; row 512 = ones -> bias grad
static B2wOp::Args args_b2w(const WS &w, int n, int *s2) {
    B2wOp::Args g{};
    g.a[0] = im2col(w.act1[0], n, 20, 20, 32, 4, 2, 9, 9);
    g.b[0] = LoadDense{w.dY2, n * 81, 64, 64};
    g.e[0] = EpiF32T{w.part2, 513, 64, 513, (size_t)64 * 513};
    const int nch = (n * 81 + 63) / 64;
    g.kc_per_split = choose_kc(nch, 5, s2);
    g.M = 513, g.N = 64, g.K = n * 81, g.splits = *s2, g.ones_at = 512, g.ones_extent = n * 81;
    return g;
}
// B2d: dY1 = relu'(x1) * transposed conv2(dY2), stride 2 split into the 4 input parity
// classes -> K = 4 taps x 64 per class instead of 16 x 64
static B2dOp::Args args_b2d(const bf16 *sh, const WS &w, int n) {
    const int tpc = (n * 100 + 127) / 128;
    B2dOp::Args g{};
    g.a[0] = tconv_p(w.dY2, n, 10, 10, 9, 9, 64, tpc);
    g.b[0] = weight_tp(sh + S_W2, 64, 4, 32, tpc);
    g.e[0] = epi_mask_p(w.dY1, w.act1[0], n, 10, 10, 32, tpc);
    g.M = 4 * tpc * 128, g.N = 32, g.K = 256, g.kc_per_split = 4, g.splits = 1, g.ones_at = -1;
    return g;
}
// B1w: dW1^T[k][o] = sum_m P1[m][k] dY1[m][o] over uint8 frames; row 256 = ones
static B1wOp::Args args_b1w(const pq_learn_args *la, const WS &w, int n, int *s1) {
    B1wOp::Args g{};
    FwdInput in{la->ring, la->records, la->idx ? la->idx : w.idx_cur, nullptr, n, REC_INTS, 0};
    g.a[0] = frames_loader(in, n);
    g.b[0] = LoadDense{w.dY1, n * 400, 32, 32};
    g.e[0] = EpiF32T{w.part1, 257, 32, 257, (size_t)32 * 257};
    const int nch = (n * 400 + 63) / 64;
    g.kc_per_split = choose_kc(nch, 3, s1, (TABLE_SAMPLES - 2) * 400 / 64);
    g.M = 257, g.N = 32, g.K = n * 400, g.splits = *s1, g.ones_at = 256, g.ones_extent = n * 400;
    return g;
}
// B4d: dY3[b][k] = relu'(x3) * sum_j W4[j][k] dh1[b][j]   (D[k][b], MN-major W4)
static int launch_b4d(const pq_net &th, int n, const WS &w, cudaStream_t st) {
    if (use_tma(n) && conv1_shift() && w.dY3p)  // unswapped, the 128-sample dh1 tile resident per CTA
        return tma_fc1_dgrad_resident(th, w.dh1_bf, w.act3[0], w.dY3, n, st, w.dY3p);
    if (use_tma(n))  // unswapped on the TMA engine: D[b][k], W4 as MN-major B
        return tma_fc1_dgrad(th, w.dh1_bf, w.act3[0], w.dY3, n, st);
    GemmArgs<LoadDense, LoadDense, EpiMaskT> g{};
    g.a[0] = LoadDense{(const bf16 *)th.shadow + S_W4, 512, 3136, 3136};
    g.b[0] = LoadDense{w.dh1_bf, n, 512, 512};
    g.e[0] = EpiMaskT{w.dY3, w.act3[0], 3136, n, 3136, w.dY3p};
    g.M = 3136, g.N = n, g.K = 512, g.kc_per_split = 8, g.splits = 1, g.ones_at = -1;
    PQ_CHECK((launch_bn<LoadDense, LoadDense, EpiMaskT, true, false, 1>(choose_bn(n), g, 1, st)), "fc1 dgrad");
    return 0;
}
static OptArgs opt_args(const pq_learn_args *la, int n, const WS &w) {
    const pq_net &th = la->theta;
    OptArgs o{};
    o.p = th.master, o.m = la->opt.m, o.v = la->opt.v;
    o.p2 = la->theta_out.master, o.m2 = la->opt_out.m, o.v2 = la->opt_out.v;
    o.shadow = (bf16 *)la->theta_out.shadow;
    o.part1 = w.part1, o.part2 = w.part2, o.part3 = w.part3, o.grad4 = nullptr;
    o.dh1 = w.dh1, o.h1 = w.h1, o.td = w.td, o.act = w.act;
    o.n = n, o.A = la->actions;
    o.lr = la->lr, o.rho = la->rho, o.kappa = la->kappa;
    o.flag = la->nonfinite, o.counter = w.upd_cur;
    o.grad_out = la->grad_out;
    o.total = n_params(la->actions);
    o.w1_perm = 1;  // both engines produce conv1's weight-gradient rows in the permuted K order
    return o;
}

// the optimizer over [lo1, hi1) u [lo2, hi2) as one part of a fused launch
struct OptOp {
    static constexpr bool GEMM = false, TABLE = false;
    static constexpr int SMEM = 0, STAGES = 1;
    static constexpr uint32_t TMEM_COLS = 32;
    using Launch = OptArgs;
    static int ctas(const OptArgs &a) { return (int)(((a.hi1 - a.lo1) + (a.hi2 - a.lo2) + 255) / 256); }
    PQ_DEV static void run(const OptArgs &a, int lin, TileRing &) {
        const int64_t t = (int64_t)lin * 256 + threadIdx.x;
        const int64_t n1 = a.hi1 - a.lo1;
        const int64_t i = t < n1 ? a.lo1 + t : a.lo2 + (t - n1);
        const bool live = t < n1 || i < a.hi2;
        const OptPre pre = live ? opt_load(a, i) : OptPre{};
        const int upd = a.counter ? *a.counter : 0;
        griddep_wait();
        griddep_launch();
        if (live) opt_param(a, i, upd, pre);
    }
};

// Single-stream learner backward (cp.async engine, PQ_FUSED, default on below batch
// 128): every launch chains to the next by PDL; the weight-gradient branch rides in
// the critical-path launches as extra CTAs:
//   B4d | {B3d, B3w, B4w+RMSProp} | {B2d, B2w} | B1w | update of all but W4
// Each part reads only what the launch before it (or older ones) wrote: B4w rewrites
// the W4 shadow after B4d read it; the update follows B3d / B2d / B1w, the last readers
// of W3 / W2 and the last producer.  The step counter advances in the head.
static bool fused_backward(int n, const pq_learn_args *la, float *grad_only) {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("PQ_FUSED");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1 && !use_tma(n) && !grad_only && n < FC_PART_MIN_BATCH;
}

// ---- the target network's forward of the NEXT step, pipelined into this step's launches
// (executor epochs, batch 32-class: pq_learn_step_pipelined).  theta-minus is fixed within
// an epoch and the head has already advanced the step counter to the next minibatch, so
// conv1 / conv2 / conv3 of the target network for step k+1 ride as extra CTAs in step k's
// fc1-dgrad, {conv2 dgrad | conv2 wgrad} and {conv1 wgrad | update} launches (each shorter
// than its host's critical tiles), and its fc1 in step k+1's conv1 launch.  Each stage
// reads what two or more launches back wrote; the same GEMM configurations as the one-shot
// forward, so the results are bit-identical.  pq_learn_target_prologue primes
// conv1..conv3 for the first step of an epoch.
// Ring depths of the small-batch critical path: every K-chunk of a tile in flight before
// its first MMA (the whole K range fits in shared memory: conv1 4 chunks of 28 KB, conv2 /
// conv3 / fc1-dgrad 8-9 of 24 / 20 KB, fc1 7 of 20 KB); one CTA per SM (grids <= 148)
// (PQ_DEEP=0: the 3-4 slot rings)
constexpr int DEEP_U8 = 6, DEEP_BN64 = 9, DEEP_BN32 = 9;
static bool deep_rings() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("PQ_DEEP");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}
template <bool D>
struct Ring {
    using F1 = GemmOp<32, false, false, D ? DEEP_U8 : 3, 1, LoadFrames, LoadDense, EpiBiasRelu>;
    using F1Late = F1;  // the target conv1 of the next step: table from the step stash
    using B4dT = GemmOp<32, true, false, D ? DEEP_BN32 : 0, 1, LoadDense, LoadDense, EpiMaskT>;     // fc1 dgrad at BN 32
    static constexpr int BN64 = D ? DEEP_BN64 : 0, BN32 = D ? DEEP_BN32 : 0;
};
using F1Op = Ring<false>::F1;
using F23Op = GemmOp<64, false, false, 0, 2, LoadIm2col, LoadDense, EpiBiasRelu>;
using F4Op = GemmOp<32, false, false, 0, 1, LoadDense, LoadDense, EpiF32T>;
static F1Op::Args args_f1(const pq_net &net, const FwdInput &in, int n, bf16 *act1) {
    F1Op::Args g{};
    g.a[0] = frames_loader(in, n);
    g.b[0] = LoadDense{(const bf16 *)net.shadow + S_W1P, 32, 256, 256};  // permuted K
    g.e[0] = EpiBiasRelu{act1, net.master + P_B1, n * 400, 32, 32, 1.0f / 255.0f};
    g.M = n * 400, g.N = 32, g.K = 256, g.kc_per_split = 4, g.splits = 1, g.ones_at = -1;
    return g;
}
static F23Op::Args args_f2(const pq_net &net, const bf16 *act1, int n, bf16 *act2) {
    F23Op::Args g{};
    g.a[0] = im2col(act1, n, 20, 20, 32, 4, 2, 9, 9);
    g.b[0] = LoadDense{(const bf16 *)net.shadow + S_W2, 64, 512, 512};
    g.e[0] = EpiBiasRelu{act2, net.master + P_B2, n * 81, 64, 64, 1.0f};
    g.M = n * 81, g.N = 64, g.K = 512, g.kc_per_split = 8, g.splits = 1, g.ones_at = -1;
    return g;
}
static F23Op::Args args_f3(const pq_net &net, const bf16 *act2, int n, bf16 *act3) {
    F23Op::Args g{};
    g.a[0] = im2col(act2, n, 9, 9, 64, 3, 1, 7, 7);
    g.b[0] = LoadDense{(const bf16 *)net.shadow + S_W3, 64, 576, 576};
    g.e[0] = EpiBiasRelu{act3, net.master + P_B3, n * 49, 64, 64, 1.0f};
    g.M = n * 49, g.N = 64, g.K = 576, g.kc_per_split = 9, g.splits = 1, g.ones_at = -1;
    return g;
}
static F4Op::Args args_f4(const pq_net &net, const bf16 *act3, int n, float *part) {
    F4Op::Args g{};
    g.a[0] = LoadDense{(const bf16 *)net.shadow + S_W4, 512, 3136, 3136};
    g.b[0] = LoadDense{act3, n, 3136, 3136};
    g.e[0] = EpiF32T{part, 512, n, 512, (size_t)n * 512};
    g.M = 512, g.N = n, g.K = 3136, g.kc_per_split = 49 / FC1_SPLITS, g.splits = FC1_SPLITS, g.ones_at = -1;
    return g;
}
static FwdInput target_input(const pq_learn_args *la) {  // next-state frames f1..f4 at *counter
    return FwdInput{la->ring, la->records, la->idx_base, la->update_counter, la->n, REC_INTS, 1};
}
static bool pipeline_ok(const pq_learn_args *la) {
    return !la->idx && la->idx_base && la->update_counter && !la->ext_targets && choose_bn(la->n) == 32 &&
           fused_backward(la->n, la, nullptr);
}

template <bool D>
static int launch_b4d_t1(const pq_learn_args *la, int n, const WS &w, cudaStream_t st) {
    using B4dTOp = typename Ring<D>::B4dT;
    using F1LateOp = typename Ring<D>::F1Late;
    const bf16 *sh = (const bf16 *)la->theta.shadow;
    typename B4dTOp::Args g{};
    g.a[0] = LoadDense{sh + S_W4, 512, 3136, 3136};
    g.b[0] = LoadDense{w.dh1_bf, n, 512, 512};
    g.e[0] = EpiMaskT{w.dY3, w.act3[0], 3136, n, 3136, w.dY3p};
    g.M = 3136, g.N = n, g.K = 512, g.kc_per_split = 8, g.splits = 1, g.ones_at = -1;
    FusedArgs<B4dTOp, F1LateOp, NoOp> f{};
    f.p0 = B4dTOp::make(g);
    // the next minibatch's frames: update id = the stash of this step's first launch + 1,
    // so the frame table and the frames are requested before the wait (the head, the
    // launch before, is what advances the live counter)
    F1Op::Args t1 = args_f1(la->target, target_input(la), n, w.act1[1]);
    t1.a[0].counter = w.step_stash;
    t1.a[0].counter_add = 1;
    f.p1 = F1LateOp::make(t1);
    f.n0 = B4dTOp::ctas(f.p0, 1), f.n1 = F1LateOp::ctas(f.p1, 1);
    // the step's update counter advance (the head's last-block bump in the other schedules):
    // this launch and the ones after it read the step's stash, never the live counter
    f.bump_src = w.step_stash, f.bump_dst = la->update_counter;
    PQ_CHECK(launch_fused(f, 0, st), "fc1 dgrad | target conv1");
    return 0;
}


// conv1 weight gradient (+ the pipelined target conv3 of the next step); the deep ring
// (7 x 32 KB: all 5 K-chunks of a split in flight) needs the launch alone on its SMs
template <bool D>
static int launch_b1w(const pq_learn_args *la, int n, const WS &w, cudaStream_t st, bool pipe, int *s1) {
    using B1 = GemmOp<64, true, true, D ? 7 : 3, 1, LoadFrames, LoadDense, EpiF32T>;  // frames before the wait
    typename B1::Launch b1 = B1::make(args_b1w(la, w, n, s1));
    if (pipe) {  // + the target conv3 of the next step
        FusedArgs<B1, F23Op, NoOp> f{};
        f.p0 = b1, f.p1 = F23Op::make(args_f3(la->target, w.act2[1], n, w.act3[1]));
        f.n0 = B1::ctas(f.p0, 1), f.n1 = F23Op::ctas(f.p1, 1);
        PQ_CHECK(launch_fused(f, 0, st), "conv1 wgrad | target conv3");
    } else {
        FusedArgs<B1, NoOp, NoOp> f{};
        f.p0 = b1;
        f.n0 = B1::ctas(f.p0, 1), f.n1 = 0;
        PQ_CHECK(launch_fused(f, 0, st), "conv1 wgrad");
    }
    return 0;
}

static int backward_fused(const pq_learn_args *la, int n, const WS &w, cudaStream_t st, bool pipe = false) {
    const pq_net &th = la->theta;
    const bf16 *sh = (const bf16 *)th.shadow;
    int s1 = 1, s2 = 1, s3 = 1;
    if (pipe) {  // fc1 dgrad + the target conv1 of the next step (its frame table after the wait:
                 // the head, the launch before, advanced the counter)
        if (int rc = deep_rings() ? launch_b4d_t1<true>(la, n, w, st) : launch_b4d_t1<false>(la, n, w, st))
            return rc;
    } else if (int rc = launch_b4d(th, n, w, st)) {
        return rc;
    }
    {  // conv3 dgrad by row-shifted descriptors over fc1 dgrad's padded copy (Dg3ShiftOp); the
       // fc1 weight gradient + RMSProp tiles start without waiting for the fc1 data gradient
       // (EpiRms4Late), so they dispatch right after the critical tiles, before the conv3
       // weight gradient (batch 32: 61.2 -> 59.4 us/step against the waiting tiles last)
        FusedArgs<Dg3ShiftOp, B4wLateOp, B3wOp> f{};
        f.p0 = Dg3ShiftOp::make(Dg3Args{w.dY3p, sh + S_W3, w.act2[0], w.dY2, n});
        f.p1 = B4wLateOp::make(args_b4w_rms<EpiRms4Late>(la, n, w));
        f.p2 = B3wOp::make(args_b3w(w, n, &s3));
        f.n0 = Dg3ShiftOp::ctas(f.p0, 1), f.n1 = B4wLateOp::ctas(f.p1, 1);
        PQ_CHECK(launch_fused(f, B3wOp::ctas(f.p2, 1), st), "conv3 dgrad | fc1 wgrad+rmsprop | conv3 wgrad");
    }
    const pq_net &tg = la->target;
    if (pipe) {  // + the target conv2 of the next step (CTAs dispatch in part order: the
                 // critical tiles, then the target stage, then the weight gradient)
        FusedArgs<B2dOp, F23Op, B2wOp> f{};
        f.p0 = B2dOp::make(args_b2d(sh, w, n));
        f.p1 = F23Op::make(args_f2(tg, w.act1[1], n, w.act2[1]));
        f.p2 = B2wOp::make(args_b2w(w, n, &s2));
        f.n0 = B2dOp::ctas(f.p0, 1), f.n1 = F23Op::ctas(f.p1, 1);
        PQ_CHECK(launch_fused(f, B2wOp::ctas(f.p2, 1), st), "conv2 dgrad | target conv2 | conv2 wgrad");
    } else {
        FusedArgs<B2dOp, B2wOp, NoOp> f{};
        f.p0 = B2dOp::make(args_b2d(sh, w, n));
        f.p1 = B2wOp::make(args_b2w(w, n, &s2));
        f.n0 = B2dOp::ctas(f.p0, 1), f.n1 = B2wOp::ctas(f.p1, 1);
        PQ_CHECK(launch_fused(f, 0, st), "conv2 dgrad | conv2 wgrad");
    }
    OptArgs o = opt_args(la, n, w);
    o.s2 = s2, o.s3 = s3;
    if (int rc = deep_rings() ? launch_b1w<true>(la, n, w, st, pipe, &s1) : launch_b1w<false>(la, n, w, st, pipe, &s1))
        return rc;
    o.s1 = s1;
    // one update launch after the conv1 weight gradient: every parameter but fc1's weight
    // (updated inside its weight-gradient GEMM); only conv1's rows wait on the launch before
    // One parameter per thread in the no-wait blocks and 4 blocks per SM: they run on the
    // SMs the conv1 weight gradient leaves free and fill the SMs as its CTAs exit, the fc
    // parameters (batch sums at small batches, the slowest) on the first threads.  Batch
    // 32: 63.3 -> 61.6 us/step against 64 blocks of 5 parameters per thread after the
    // conv1 blocks (PQ_OPT_TAIL=64,0,1).
    static int nb2 = -1, first1 = 2, minb = 2;
    if (nb2 < 0) {  // PQ_OPT_TAIL=nb2,first1,minblocks (A/B)
        nb2 = 320;
        if (const char *e = getenv("PQ_OPT_TAIL")) sscanf(e, "%d,%d,%d", &nb2, &first1, &minb);
    }
    const int nb1 = (int)((P_W2 - P_W1 + 255) / 256);
    const int pt = (int)((P_W4 - P_W2 + o.total - P_B4 + nb2 * 256 - 1) / (nb2 * 256));
    auto kern = minb >= 4 ? k_opt_tail<4> : minb >= 3 ? k_opt_tail<3> : minb >= 2 ? k_opt_tail<2> : k_opt_tail<1>;
    PQ_CHECK(launch_k(kern, dim3((unsigned)(nb1 + nb2)), dim3(256), 0, st, o, nb1, pt, first1), "optimizer");
    return 0;
}

// grad_only != NULL: write the summed gradient of every parameter there instead of
// updating theta / opt (the data-parallel learner all-reduces it, then pq_rmsprop_apply)
// fc1_done (grad_only): recorded once grad_only[P_W4, P_B4) -- the fc1 weight gradient, 95%
// of the bytes -- is complete, so its all-reduce can start under the conv backward
static int backward_and_update(const pq_learn_args *la, int n, const WS &w, cudaStream_t st,
                               float *grad_only = nullptr, cudaEvent_t fc1_done = nullptr) {
    if (fused_backward(n, la, grad_only)) return backward_fused(la, n, w, st);
    const pq_net &th = la->theta;
    const bf16 *sh = (const bf16 *)th.shadow;
    int s1 = 1, s2 = 1, s3 = 1;
    Fork *fk = nullptr;
    if (int rc = get_fork(&fk)) return rc;
    cudaStream_t side = fk->side, side2 = fk->side2;
    if (int rc = launch_b4d(th, n, w, st)) return rc;
    // fork after the fc1 data gradient: the fused fc1 update below rewrites the W4
    // shadow that B4d reads, so it must not start earlier
    PQ_CHECK(cudaEventRecord(fk->ev[1], st), "fork1");
    PQ_CHECK(cudaStreamWaitEvent(side, fk->ev[1], 0), "fork1 wait");
    PQ_CHECK(cudaStreamWaitEvent(side2, fk->ev[1], 0), "fork1 wait 2");
    // large batches: the fc2 / fc1-bias batch sums as chunk partials on the wgrad branch
    // (the optimizer then reduces n/64 partials per parameter instead of n samples)
    const int fc_chunks = n >= FC_PART_MIN_BATCH ? (n + FC_CHUNK - 1) / FC_CHUNK : 0;
    if (fc_chunks) {
        static bool configured = false;
        if (!configured) {
            PQ_CHECK(cudaFuncSetAttribute(k_fc2_partials, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          MAX_ACTIONS * 512 * 4),
                     "fc2 partials smem");
            configured = true;
        }
    }
    if (fc_chunks)
        PQ_CHECK(launch_k(k_fc2_partials, dim3(fc_chunks), dim3(512), (size_t)la->actions * 512 * 4, side2,
                          (const float *)w.h1,
                          (const float *)w.dh1, (const float *)w.td, (const int32_t *)w.act, n, la->actions,
                          w.fcpart),
                 "fc2 partials");
    if (grad_only) {  // B4w: dW4[j][k] = sum_b dh1[b][j] x3[b][k] -> grad (row-major = param order)
        GemmArgs<LoadDense, LoadDense, EpiF32> g{};
        g.a[0] = LoadDense{w.dh1T, 512, n, w.n8};
        g.b[0] = LoadDense{w.act3[0], n, 3136, 3136};
        g.e[0] = EpiF32{grad_only + P_W4, 512, 3136, 3136, 0};
        g.M = 512, g.N = 3136, g.K = n, g.kc_per_split = (n + 63) / 64, g.splits = 1, g.ones_at = -1;
        PQ_CHECK((launch_gemm<64, false, true, 4>(g, 1, side)), "fc1 wgrad");
        if (fc1_done) PQ_CHECK(cudaEventRecord(fc1_done, side), "fc1 gradient event");
    } else {  // (the cp.async engine: its staged RMSProp epilogue walks the tile with all 8 warps)
        PQ_CHECK((launch_gemm<128, false, true, 4>(args_b4w_rms<EpiRms>(la, n, w), 1, side)), "fc1 wgrad+rmsprop");
    }
    {
        B3wOp::Args g = args_b3w(w, n, &s3);
        if (use_tma(n)) {
            if (int rc = tma_conv3_wgrad(w.act2[0], w.dY3, w.part3, g.kc_per_split, s3, n, side2)) return rc;
        } else {
            PQ_CHECK((launch_gemm<64, true, true>(g, 1, side2)), "conv3 wgrad");
        }
    }
    const bool shift = conv1_shift() && w.dY1p && w.dY2p;  // shifted-descriptor conv kernels (TMA engine)
    if (use_tma(n) && shift && w.dY3p) {  // over fc1's data gradient on the padded 11 x 11 grid
        if (int rc = tma_conv3_dgrad_shift(th, w.dY3p, w.act2[0], w.dY2, w.dY2p, w.dY2q, n, st)) return rc;
    } else if (use_tma(n)) {
        if (int rc = tma_conv3_dgrad(th, w.dY3, w.act2[0], w.dY2, n, st, shift ? w.dY2p : nullptr,
                                     shift ? w.dY2q : nullptr))
            return rc;
    } else {
        PQ_CHECK((launch_gemm<64, false, true, 0, 2>(args_b3d(sh, w, n), 1, st)), "conv3 dgrad");
    }
    PQ_CHECK(cudaEventRecord(fk->ev[2], st), "fork2");
    PQ_CHECK(cudaStreamWaitEvent(side2, fk->ev[2], 0), "fork2 wait");
    if (shift) {  // over act1's space-to-depth copy and dY2 on the 10 x 10 grid
        const int nk = (n * 100 + 63) / 64, kc = (nk + MAX_SPLITS - 1) / MAX_SPLITS;
        s2 = (nk + kc - 1) / kc;
        if (int rc = tma_conv2_wgrad_shift(w.act1s2[0], w.dY2q, w.part2, kc, s2, n, side2)) return rc;
    } else {
        PQ_CHECK((launch_gemm<64, true, true>(args_b2w(w, n, &s2), 1, side2)), "conv2 wgrad");
    }
    if (use_tma(n)) {
        if (shift) {  // dY1 onto the padded grid of the shifted conv1 weight gradient
            if (int rc = tma_conv2_dgrad_shift(th, w.dY2p, w.act1s2[0], w.dY1p, n, 1, st, 1)) return rc;
        } else if (int rc = tma_conv2_dgrad(th, w.dY2, w.act1[0], w.dY1, n, st, 0)) {
            return rc;
        }
    } else {
        PQ_CHECK((launch_gemm<64, false, true, 0, 2>(args_b2d(sh, w, n), 1, st)), "conv2 dgrad");
    }
    OptArgs o = opt_args(la, n, w);
    if (fc_chunks) o.fcpart = w.fcpart, o.fcchunks = fc_chunks;
    {
        B1wOp::Args g = args_b1w(la, w, n, &s1);
        if (use_tma(n) && w.s2d) {  // over the space-to-depth stacks
            const int nframes = la->ext_targets ? 4 : 5;
            if (shift) {
                const int nk = (n * 441 + 63) / 64, kc = (nk + P1_MAX_SPLITS - 1) / P1_MAX_SPLITS;
                s1 = (nk + kc - 1) / kc;  // one CTA per split, all three M tiles
                if (int rc = tma_conv1_wgrad_shift(w.s2d, nframes, w.dY1p, w.part1, kc, s1, n, st)) return rc;
            } else if (int rc = tma_conv1_wgrad(w.s2d, nframes, w.dY1, w.part1, g.kc_per_split, s1, n, st)) {
                return rc;
            }
        } else {
            PQ_CHECK((launch_gemm<64, true, true>(g, 1, st)), "conv1 wgrad");
        }
    }
    // join the weight-gradient branch
    PQ_CHECK(cudaEventRecord(fk->ev[3], side), "join");
    PQ_CHECK(cudaEventRecord(fk->ev[4], side2), "join 2");
    PQ_CHECK(cudaStreamWaitEvent(st, fk->ev[3], 0), "join wait");
    PQ_CHECK(cudaStreamWaitEvent(st, fk->ev[4], 0), "join wait 2");
    if (!grad_only) {  // every parameter but fc1's weight, after the join
        o.s1 = s1, o.s2 = s2, o.s3 = s3;
        o.lo1 = P_W1, o.hi1 = P_W4, o.lo2 = P_B4, o.hi2 = o.total;
        if (!la->idx && la->update_counter) o.bump = la->update_counter, o.bump_done = w.done;
        const int64_t cnt = P_W4 + (o.total - P_B4);
        PQ_CHECK(launch_k(k_optimizer, dim3((unsigned)((cnt + 255) / 256)), dim3(256), 0, st, o), "optimizer");
    }
    if (grad_only) {
        o.s1 = s1, o.s2 = s2, o.s3 = s3;
        o.grad_out = grad_only;
        const int64_t cnt = P_W4 + (o.total - P_B4);
        PQ_CHECK(launch_k(k_grad_only, dim3((unsigned)((cnt + 255) / 256)), dim3(256), 0, st, o), "gradient");
    }
    return 0;
}

// ------------------------------------------------------------------ misc kernels
__global__ void k_f32_to_bf16(const float *src, bf16 *dst, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __float2bfloat16_rn(src[i]);
}
__global__ void k_w1_perm(const float *w1, bf16 *dst) {  // dst[o][w1_perm(k)] = w1[o][k]
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 8192) dst[(i >> 8) * 256 + w1_perm(i & 255)] = __float2bfloat16_rn(w1[i]);
}

__global__ void k_rmsprop(const float *p, const float *g, const float *m, const float *v,
                          int64_t n, float lr, float rho, float kappa, float *p2, float *m2,
                          float *v2, int32_t *flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float gi = g[i];
    if (!isfinite(gi) && flag) atomicMin(flag, 0);
    float mi = rho * m[i] + (1.0f - rho) * gi;
    float vi = rho * v[i] + (1.0f - rho) * gi * gi;
    m2[i] = mi;
    v2[i] = vi;
    p2[i] = p[i] - lr * gi / sqrtf(vi - mi * mi + kappa);
}

// acting forward: F1..F4 over the W current stacks (refs [W][4]), fc1 partials out
int act_forward(pq_net net, const uint8_t *ring, const int32_t *stack, int W, int A, void *ws,
                int max_batch, const float **part_out, uint32_t **done_out, int *splits_out, cudaStream_t st) {
    WS w = carve(ws, max_batch, A);
    FwdInput in{ring, stack, nullptr, nullptr, 0, 4, 0};
    int rc = forward_gemms(&net, &in, 1, W, w, st);
    *part_out = w.fc1part[0];
    *done_out = w.done + 1;
    *splits_out = fc1_splits(W, 1);
    return rc;
}

// online conv1 (+ the target fc1 of this step) .. fc1 of the pipelined step
template <bool D>
static int forward_pipelined(const pq_learn_args *la, const FwdInput &in, int n, const WS &w, cudaStream_t st) {
    using F1T = typename Ring<D>::F1;
    {
        FusedArgs<F1T, F4Op, NoOp> f{};
        f.p0 = F1T::make(args_f1(la->theta, in, n, w.act1[0]));
        f.p1 = F4Op::make(args_f4(la->target, w.act3[1], n, w.fc1part[1]));
        f.n0 = F1T::ctas(f.p0, 1), f.n1 = F4Op::ctas(f.p1, 1);
        f.stash_src = la->update_counter, f.stash_dst = w.step_stash;
        PQ_CHECK(launch_fused(f, 0, st), "conv1 | target fc1");
    }
    PQ_CHECK((launch_gemm<64, false, false, Ring<D>::BN64, 2>(args_f2(la->theta, w.act1[0], n, w.act2[0]), 1, st)),
             "conv2 forward");
    PQ_CHECK((launch_gemm<64, false, false, Ring<D>::BN64, 2>(args_f3(la->theta, w.act2[0], n, w.act3[0]), 1, st)),
             "conv3 forward");
    PQ_CHECK((launch_gemm<32, false, false, Ring<D>::BN32, 1>(args_f4(la->theta, w.act3[0], n, w.fc1part[0]), 1, st)),
             "fc1 forward");
    return 0;
}

}  // namespace pq

using namespace pq;

// ------------------------------------------------------------------ C ABI
extern "C" {

int pq_abi_version(void) { return PQ_ABI_VERSION; }

int pq_fc1_splits(int n, int groups) { return fc1_splits(n, groups); }

int pq_cta_trace(int on, unsigned long long *out, int *count) {
    if (out) {
        static CtaTrace h;
        PQ_CHECK(cudaMemcpyFromSymbol(&h, g_ct, sizeof(CtaTrace)), "cta trace read");
        *count = h.n < 8192 ? (int)h.n : 8192;
        memcpy(out, h.r, sizeof(h.r));
    }
    static CtaTrace z;
    memset(&z, 0, sizeof(z));
    z.on = on;
    PQ_CHECK(cudaMemcpyToSymbol(g_ct, &z, sizeof(CtaTrace)), "cta trace reset");
    return 0;
}

int pq_timeline(int on, unsigned long long *out, int *count) {
    if (out) {
        static Timeline h;
        PQ_CHECK(cudaMemcpyFromSymbol(&h, g_tl, sizeof(Timeline)), "timeline read");
        *count = h.n < 256 ? h.n : 256;
        memcpy(out, h.t, sizeof(h.t));
    }
    static Timeline z;
    memset(&z, 0, sizeof(z));
    z.on = on;
    PQ_CHECK(cudaMemcpyToSymbol(g_tl, &z, sizeof(Timeline)), "timeline reset");
    return 0;
}
const char *pq_last_error(void) { return g_err; }
int64_t pq_num_params(int actions) { return n_params(actions); }
int64_t pq_num_shadow(void) { return S_TOTAL; }

size_t pq_workspace_bytes(int max_batch, int actions) {
    return carve(nullptr, max_batch, actions).bytes;
}

int pq_workspace_layout(int max_batch, int actions, int64_t *offsets) {
    char *base = reinterpret_cast<char *>(size_t(1) << 40);
    WS w = carve(base, max_batch, actions);
    const void *ptrs[] = {w.act1[0], w.act2[0], w.act3[0], w.fc1part[0], w.act1[1], w.act2[1],
                          w.act3[1], w.fc1part[1], w.q, w.h1, w.dh1, w.td, w.dh1_bf, w.dh1T,
                          w.act, w.dY3, w.dY2, w.dY1, w.part1, w.part2, w.part3, w.grad4, w.dY1p, w.dY2p,
                          w.act1s2[0], w.act1s2[1]};
    for (int i = 0; i < 26; ++i) offsets[i] = ptrs[i] ? (const char *)ptrs[i] - base : -1;
    return 0;
}

int pq_l2_persist(void *stream, const void *base, size_t bytes, float hit_ratio) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaStreamAttrValue v{};
    if (bytes && base) {
        int dev = 0, max_persist = 0, max_window = 0;
        PQ_CHECK(cudaGetDevice(&dev), "device");
        PQ_CHECK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev), "persisting L2 size");
        PQ_CHECK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev), "window size");
        const size_t set_aside = bytes < (size_t)max_persist ? bytes : (size_t)max_persist;
        PQ_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside), "persisting L2 limit");
        const size_t win = bytes < (size_t)max_window ? bytes : (size_t)max_window;
        v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
        v.accessPolicyWindow.num_bytes = win;
        // hit ratio scaled so the persisting lines fit the set-aside
        const float fit = (float)set_aside / (float)win;
        v.accessPolicyWindow.hitRatio = hit_ratio < fit ? hit_ratio : fit;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
        v.accessPolicyWindow.num_bytes = 0;
    }
    PQ_CHECK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v), "access policy window");
    return 0;
}

int pq_net_sync_shadow(pq_net net, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t src_off[4] = {P_W1, P_W2, P_W3, P_W4};
    const int64_t dst_off[4] = {S_W1, S_W2, S_W3, S_W4};
    const int64_t cnt[4] = {8192, 32768, 36864, 1605632};
    for (int l = 0; l < 4; ++l) {
        k_f32_to_bf16<<<(unsigned)((cnt[l] + 255) / 256), 256, 0, st>>>(
            net.master + src_off[l], (bf16 *)net.shadow + dst_off[l], cnt[l]);
    }
    k_w1_perm<<<32, 256, 0, st>>>(net.master + P_W1, (bf16 *)net.shadow + S_W1P);
    return cuda_err(cudaGetLastError(), "sync_shadow");
}

int pq_net_copy(pq_net dst, pq_net src, int actions, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    PQ_CHECK(cudaMemcpyAsync(dst.master, src.master, n_params(actions) * 4,
                             cudaMemcpyDeviceToDevice, st), "net_copy master");
    PQ_CHECK(cudaMemcpyAsync(dst.shadow, src.shadow, S_TOTAL * 2, cudaMemcpyDeviceToDevice, st),
             "net_copy shadow");
    return 0;
}

int pq_forward(pq_net net, const uint8_t *ring, const int32_t *refs, const int64_t *map,
               int ref_stride, int ref_off, int n, int actions, float *q_out, void *ws,
               int max_batch, void *stream) {
    if (n < 1 || n > max_batch) return set_err("batch size out of range for the workspace");
    if (actions < 1 || actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    cudaStream_t st = (cudaStream_t)stream;
    WS w = carve(ws, max_batch, actions);
    FwdInput in{ring, refs, map, nullptr, 0, ref_stride, ref_off};
    int rc = forward_gemms(&net, &in, 1, n, w, st);
    if (rc) return rc;
    rc = head(&net, 1, n, actions, w, 0, nullptr, st);
    if (rc) return rc;
    if (q_out)
        PQ_CHECK(cudaMemcpyAsync(q_out, w.q, (size_t)n * actions * 4, cudaMemcpyDeviceToDevice, st),
                 "forward q copy");
    return 0;
}

int pq_learn_step(const pq_learn_args *la, void *stream) {
    const int n = la->n;
    if (n < 1 || n > la->max_batch) return set_err("batch size out of range for the workspace");
    if (la->actions < 1 || la->actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    cudaStream_t st = (cudaStream_t)stream;
    WS w = carve(la->ws, la->max_batch, la->actions);
    const int64_t *map = la->idx ? la->idx : la->idx_base;
    const int32_t *counter = la->idx ? nullptr : la->update_counter;
    pq_net nets[2] = {la->theta, la->target};
    FwdInput ins[2] = {{la->ring, la->records, map, counter, n, REC_INTS, 0},
                       {la->ring, la->records, map, counter, n, REC_INTS, 1}};
    const int groups = la->ext_targets ? 1 : 2;
    int rc = forward_gemms(nets, ins, groups, n, w, st, true);
    if (rc) return rc;
    rc = head(nets, groups, n, la->actions, w, 1, la, st, fused_backward(n, la, nullptr));
    if (rc) return rc;
    return backward_and_update(la, n, w, st);
}

// One learner step with the target forward pipelined (see backward_fused): the online
// conv1 launch also runs the target fc1 of this step (its conv3 output came from the
// previous step or the prologue); then online conv2..fc1, the head, the backward.
int pq_learn_step_pipelined(const pq_learn_args *la, void *stream) {
    const int n = la->n;
    if (n < 1 || n > la->max_batch) return set_err("batch size out of range for the workspace");
    if (la->actions < 1 || la->actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    if (!pipeline_ok(la)) return pq_learn_step(la, stream);
    cudaStream_t st = (cudaStream_t)stream;
    WS w = carve(la->ws, la->max_batch, la->actions);
    const pq_net nets[2] = {la->theta, la->target};
    const FwdInput in{la->ring, la->records, la->idx_base, la->update_counter, n, REC_INTS, 0};
    if (int rc = deep_rings() ? forward_pipelined<true>(la, in, n, w, st) : forward_pipelined<false>(la, in, n, w, st))
        return rc;
    // the update counter advances in the fc1 data-gradient launch (launch_b4d_t1), not the head
    if (int rc = head(nets, 2, n, la->actions, w, 1, la, st, false)) return rc;
    return backward_fused(la, n, w, st, true);
}

// Target conv1..conv3 of the minibatch at *update_counter (the first step of an epoch,
// after theta-minus and the index table changed): primes pq_learn_step_pipelined.
int pq_learn_target_prologue(const pq_learn_args *la, void *stream) {
    if (!pipeline_ok(la)) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int n = la->n;
    WS w = carve(la->ws, la->max_batch, la->actions);
    const pq_net &tg = la->target;
    PQ_CHECK((launch_gemm<32, false, false, 3, 1>(args_f1(tg, target_input(la), n, w.act1[1]), 1, st)),
             "target conv1 (prologue)");
    PQ_CHECK((launch_gemm<64, false, false, 0, 2>(args_f2(tg, w.act1[1], n, w.act2[1]), 1, st)),
             "target conv2 (prologue)");
    PQ_CHECK((launch_gemm<64, false, false, 0, 2>(args_f3(tg, w.act2[1], n, w.act3[1]), 1, st)),
             "target conv3 (prologue)");
    return 0;
}

int pq_learn_grad(const pq_learn_args *la, float *grad, void *stream) { return pq_learn_grad_ev(la, grad, stream, nullptr); }

int pq_learn_grad_ev(const pq_learn_args *la, float *grad, void *stream, void *fc1_done) {
    const int n = la->n;
    if (n < 1 || n > la->max_batch) return set_err("batch size out of range for the workspace");
    if (la->actions < 1 || la->actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    if (!grad) return set_err("gradient buffer required");
    cudaStream_t st = (cudaStream_t)stream;
    WS w = carve(la->ws, la->max_batch, la->actions);
    const int64_t *map = la->idx ? la->idx : la->idx_base;
    const int32_t *counter = la->idx ? nullptr : la->update_counter;
    pq_net nets[2] = {la->theta, la->target};
    FwdInput ins[2] = {{la->ring, la->records, map, counter, n, REC_INTS, 0},
                       {la->ring, la->records, map, counter, n, REC_INTS, 1}};
    const int groups = la->ext_targets ? 1 : 2;
    int rc = forward_gemms(nets, ins, groups, n, w, st, true);
    if (rc) return rc;
    rc = head(nets, groups, n, la->actions, w, 1, la, st, false);
    if (rc) return rc;
    return backward_and_update(la, n, w, st, grad, (cudaEvent_t)fc1_done);
}

int pq_rmsprop_apply(pq_net theta, pq_opt opt, const float *grad, int actions, float lr, float rho,
                     float kappa, int32_t *nonfinite, int update_id, void *stream) {
    if (actions < 1 || actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    const int64_t total = n_params(actions);
    k_rmsprop_apply<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        theta.master, opt.m, opt.v, (bf16 *)theta.shadow, grad, total, lr, rho, kappa, nonfinite, update_id);
    return cuda_err(cudaGetLastError(), "rmsprop_apply");
}

int pq_rmsprop_f32(const float *p, const float *g, const float *m, const float *v, int64_t n,
                   float lr, float rho, float kappa, float *p2, float *m2, float *v2,
                   int32_t *nonfinite, void *stream) {
    k_rmsprop<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        p, g, m, v, n, lr, rho, kappa, p2, m2, v2, nonfinite);
    return cuda_err(cudaGetLastError(), "rmsprop");
}

uint64_t pq_theta_hash_f64(const double *x, int64_t n) {
    uint64_t h = 0xCBF29CE484222325ULL;
    const unsigned char *b = reinterpret_cast<const unsigned char *>(x);
    for (int64_t i = 0; i < n * 8; ++i) {
        h ^= b[i];
        h *= 0x100000001B3ULL;
    }
    return h;
}

uint64_t pq_theta_hash_f32(const float *x, int64_t n) {
    uint64_t h = 0xCBF29CE484222325ULL;
    for (int64_t i = 0; i < n; ++i) {
        double d = (double)x[i];
        unsigned char b[8];
        memcpy(b, &d, 8);
        for (int k = 0; k < 8; ++k) {
            h ^= b[k];
            h *= 0x100000001B3ULL;
        }
    }
    return h;
}

}  // extern "C"
