// Persistent DQN learner: many learner steps (agent.train_minibatch, agent.py:84-105)
// in ONE launch of one 256-thread CTA per SM.
//
// A batch-32 step is ~2 GFLOP spread over ten dependent GEMM-shaped stages; as separate
// launches it is a chain of launch / drain / TMEM-allocation latencies with the tensor
// pipe idle >95% of the time (profiles/r1_v9_summary.md).  Here every CTA keeps its
// TMEM accumulator, operand ring and mbarriers for the whole launch and the stages
// become PHASES separated by a grid barrier.  Each phase is a list of jobs (GEMM tiles,
// head samples, optimizer slices) dealt round-robin to the CTAs; work that is not on
// the critical chain rides in the idle CTAs of other phases:
//   * the target-network forward of step u+1 (theta-minus and the epoch's sample
//     indices are fixed during the launch) runs in phases 1-4 of step u;
//   * the fc1 weight gradient + fused RMSProp (196 tiles, the only HBM-heavy stage) is
//     spread over phases 6-9 of step u and 0-2 of step u+1 (act3 is double-buffered by
//     step parity; it must finish before step u+1's fc1 forward reads the new W4);
//   * the small-layer RMSProp slices run where their gradients are complete and before
//     their weights are next read.
// Phase plan of step u (critical job first, fillers after):
//   P0 F1 online conv1            | fc1 wgrad+RMS (u-1)
//   P1 F2 online conv2            | F1 target (u+1) | fc1 wgrad+RMS (u-1)
//   P2 F3 online conv3            | F2 target (u+1) | fc1 wgrad+RMS (u-1)
//   P3 F4 online fc1 (split-K)    | F3 target (u+1)
//   P4 head (fc2, TD target, delta, fc2 back-prop) | F4 target (u+1)
//   P5 fc1 dgrad                  | fc2 / fc1-bias RMSProp
//   P6 conv3 dgrad, conv3 wgrad   | fc1 wgrad+RMS
//   P7 conv2 dgrad, conv2 wgrad   | fc1 wgrad+RMS
//   P8 conv1 wgrad                | fc1 wgrad+RMS
//   P9 conv1/conv2/conv3 RMSProp  | fc1 wgrad+RMS
// The arithmetic of every job is the one-shot path's (same loaders, epilogues, head and
// optimizer functions), so the two agree to fp32 split-K summation order.
#include <algorithm>
#include <cstring>

#include "../../include/paraq_b200.h"
#include "learn_parts.cuh"

namespace pq {
int set_err(const char *msg);
int cuda_err(cudaError_t e, const char *where);
#define PQ_CUDA_TRY(expr)                        \
    do {                                         \
        int _rc = cuda_err((expr), #expr);       \
        if (_rc) return _rc;                     \
    } while (0)

constexpr int PL_STAGES = 6;
constexpr int PL_SLOT = 32 * 1024;  // A 16 KB + B (BN = 64) 8 KB + uint8 staging 8 KB
constexpr int PL_SMEM = PL_STAGES * PL_SLOT + 1024;
constexpr int PL_FC1_KC = 3;  // fc1 forward: 49 K-chunks in 17 splits
constexpr int PL_FC1_SPLITS = (49 + PL_FC1_KC - 1) / PL_FC1_KC;
constexpr int PL_OPT_PER_JOB = 1024;  // parameters per optimizer job (4 per thread)

enum Job : int16_t {
    J_F1, J_F2, J_F3, J_F4, J_HEAD, J_B4D, J_OPT_FC2, J_B3D, J_B3W, J_B4W, J_B2D, J_B2W,
    J_OPT_C3, J_B1W, J_OPT_C2, J_OPT_C1, J_COUNT
};

struct Seg {
    int16_t type;
    int8_t grp;  // 0 online, 1 target (forward jobs)
    int8_t du;   // step offset of the job relative to the running step (-1, 0, +1)
    int32_t begin, end;
};
constexpr int PL_MAX_PHASES = 12, PL_MAX_SEGS = 6;
struct PhasePlan {
    int nseg;
    Seg seg[PL_MAX_SEGS];
};
struct Sched {
    int nphases;
    PhasePlan ph[PL_MAX_PHASES];
};
enum { SCHED_PROLOGUE = 0, SCHED_STEADY = 1, SCHED_LAST = 2 };

struct PLearnArgs {
    pq_net theta, target;
    pq_opt opt;
    const uint8_t *ring;
    const int32_t *records;
    const int64_t *idx_base;  // [updates][n] epoch index table
    int32_t *update_counter;  // first step id of the launch; += n_updates at the end
    int n, A, n8, n_updates;
    float gamma, lr, rho, kappa;
    int32_t *nonfinite;
    float *grad_out, *q_out, *td_out;  // optional (values of the last step)
    // workspace
    bf16 *act1[2], *act2[2], *act3[2][2];
    float *fc1part[2][2];
    float *q, *h1, *dh1, *td;
    bf16 *dh1_bf, *dh1T;
    int32_t *act;
    bf16 *dY3, *dY2, *dY1;
    float *part1, *part2, *part3;
    int s1, s2, s3, kc1, kc2, kc3;
    unsigned *bar;
    unsigned long long *trace;  // optional [phases run][gridDim][2] (jobs done, barrier passed) ns
    Sched sched[3];
};

// ------------------------------------------------------------------ job counts
struct Counts {
    int t1, t2, t3, f4_nt, b4_nt, tpc;
};
__host__ __device__ inline Counts counts_of(int n) {
    Counts c;
    c.t1 = (n * 400 + 127) / 128;
    c.t2 = (n * 81 + 127) / 128;
    c.t3 = (n * 49 + 127) / 128;
    c.f4_nt = (n + 63) / 64;
    c.b4_nt = (n + 63) / 64;
    c.tpc = (n * 100 + 127) / 128;
    return c;
}
__host__ __device__ inline int64_t opt_lo(int type) {
    return type == J_OPT_C1 ? P_W1 : type == J_OPT_C2 ? P_W2 : type == J_OPT_C3 ? P_W3 : P_B4;
}
__host__ __device__ inline int64_t opt_hi(int type, int A) {
    return type == J_OPT_C1 ? P_W2 : type == J_OPT_C2 ? P_W3 : type == J_OPT_C3 ? P_W4 : n_params(A);
}
__host__ __device__ inline int njobs(int type, int n, int A, int s1, int s2, int s3) {
    const Counts c = counts_of(n);
    switch (type) {
        case J_F1: return c.t1;
        case J_F2: return c.t2;
        case J_F3: return c.t3;
        case J_F4: return 4 * c.f4_nt * PL_FC1_SPLITS;
        case J_HEAD: return n;
        case J_B4D: return 25 * c.b4_nt;
        case J_B3D: return c.t2;
        case J_B3W: return 5 * s3;
        case J_B4W: return 4 * 49;
        case J_B2D: return 4 * c.tpc;
        case J_B2W: return 5 * s2;
        case J_B1W: return 3 * s1;
        default: return (int)((opt_hi(type, A) - opt_lo(type) + PL_OPT_PER_JOB - 1) / PL_OPT_PER_JOB);
    }
}

// ------------------------------------------------------------------ grid barrier
// Monotonic arrival counter (zeroed before the launch); the k-th barrier completes when
// it reaches k * gridDim.x.  Release / acquire at gpu scope (the fences also invalidate
// the SM's L1 so later plain loads see other CTAs' writes).
PQ_DEV void grid_barrier(unsigned *bar, unsigned &target) {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// ------------------------------------------------------------------ jobs
struct Ctx {
    const PLearnArgs *a;
    TileRing *R;
    int u_base;
};

template <int BN, bool AMN, bool BMN, class LA, class LB, class EP>
PQ_DEV void tile(const Ctx &c, const LA &la, const LB &lb, const EP &ep, int kb0, int kb1, int m0,
                 int n0, int split = 0, int ones_at = -1, int ones_extent = 0) {
    gemm_tile<BN, AMN, BMN, PL_STAGES, PL_SLOT, 0>(la, lb, ep, kb0, kb1, m0, n0, split, ones_at,
                                                   ones_extent, *c.R, NoHook{});
}

PQ_DEV void run_job(const Ctx &c, int type, int g, int uj, int j) {
    const PLearnArgs &a = *c.a;
    const int n = a.n, par = uj & 1;
    const int upd = c.u_base + uj;
    const int64_t *map = a.idx_base + (int64_t)upd * n;
    const pq_net &net = g ? a.target : a.theta;
    const bf16 *sh = (const bf16 *)net.shadow;
    const bf16 *tsh = (const bf16 *)a.theta.shadow;
    switch (type) {
        case J_F1: {  // conv1 8x8/4 over the uint8 frame stacks, bias + ReLU, x 1/255
            tile<32, false, false>(c, frames(a.ring, a.records, map, nullptr, 0, n, REC_INTS, g),
                                   LoadDense{sh + S_W1, 32, 256, 256},
                                   EpiBiasRelu{a.act1[g], net.master + P_B1, n * 400, 32, 32, 1.0f / 255.0f},
                                   0, 4, j * 128, 0);
            break;
        }
        case J_F2:
            tile<64, false, false>(c, im2col(a.act1[g], n, 20, 20, 32, 4, 2, 9, 9),
                                   LoadDense{sh + S_W2, 64, 512, 512},
                                   EpiBiasRelu{a.act2[g], net.master + P_B2, n * 81, 64, 64, 1.0f}, 0, 8,
                                   j * 128, 0);
            break;
        case J_F3:
            tile<64, false, false>(c, im2col(a.act2[g], n, 9, 9, 64, 3, 1, 7, 7),
                                   LoadDense{sh + S_W3, 64, 576, 576},
                                   EpiBiasRelu{a.act3[g][par], net.master + P_B3, n * 49, 64, 64, 1.0f}, 0, 9,
                                   j * 128, 0);
            break;
        case J_F4: {  // fc1 swapped: D[j][b] = W4[j] . x[b], split-K partials [s][b][j]
            const Counts cn = counts_of(n);
            const int mt = j & 3, r = j >> 2, nt = r % cn.f4_nt, sp = r / cn.f4_nt;
            const int kb0 = sp * PL_FC1_KC, kb1 = min(49, kb0 + PL_FC1_KC);
            tile<64, false, false>(c, LoadDense{sh + S_W4, 512, 3136, 3136},
                                   LoadDense{a.act3[g][par], n, 3136, 3136},
                                   EpiF32T{a.fc1part[g][par], 512, n, 512, (size_t)n * 512}, kb0, kb1,
                                   mt * 128, nt * 64, sp);
            break;
        }
        case J_HEAD: {
            HeadArgs h{};
            h.part[0] = a.fc1part[0][par], h.part[1] = a.fc1part[1][par];
            h.master[0] = a.theta.master, h.master[1] = a.target.master;
            h.groups = 2, h.n = n, h.A = a.A, h.n8 = a.n8;
            h.records = a.records, h.idx = map;
            h.gamma = a.gamma, h.learner = 1;
            h.q_out = a.q, h.h1 = a.h1, h.dh1 = a.dh1, h.td = a.td, h.dh1_bf = a.dh1_bf, h.dh1T = a.dh1T;
            h.act_out = a.act, h.q_copy = a.q_out, h.td_copy = a.td_out;
            head_sample<PL_FC1_SPLITS>(h, j);
            __syncthreads();  // head shared memory is reused by the next job
            break;
        }
        case J_B4D: {  // dY3[b][k] = relu'(x3) * sum_j W4[j][k] dh1[b][j]  (D[k][b], MN-major W4)
            const int mt = j % 25, nt = j / 25;
            tile<64, true, false>(c, LoadDense{tsh + S_W4, 512, 3136, 3136}, LoadDense{a.dh1_bf, n, 512, 512},
                                  EpiMaskT{a.dY3, a.act3[0][par], 3136, n, 3136}, 0, 8, mt * 128, nt * 64);
            break;
        }
        case J_B3D:  // dY2 = relu'(x2) * transposed conv3(dY3)
            tile<64, false, true>(c, tconv(a.dY3, n, 9, 9, 7, 7, 64, 3), weight_t(tsh + S_W3, 64, 3, 64),
                                  EpiMask{a.dY2, a.act2[0], n * 81, 64, 64}, 0, 9, j * 128, 0);
            break;
        case J_B3W: {  // dW3^T[k][o] = sum_m P3[m][k] dY3[m][o]; row 576 = ones -> bias
            const int mt = j % 5, sp = j / 5;
            const int nch = (n * 49 + 63) / 64, kb0 = sp * a.kc3, kb1 = min(nch, kb0 + a.kc3);
            tile<64, true, true>(c, im2col(a.act2[0], n, 9, 9, 64, 3, 1, 7, 7), LoadDense{a.dY3, n * 49, 64, 64},
                                 EpiF32T{a.part3, 577, 64, 577, (size_t)64 * 577}, kb0, kb1, mt * 128, 0, sp,
                                 576, n * 49);
            break;
        }
        case J_B4W: {  // dW4[j][k] = sum_b dh1[b][j] x3[b][k] with centered RMSProp in the epilogue
            const int mt = j & 3, nt = j >> 2;
            EpiRms e{};
            e.p = a.theta.master, e.m = a.opt.m, e.v = a.opt.v;
            e.p2 = a.theta.master, e.m2 = a.opt.m, e.v2 = a.opt.v;
            e.shadow = (bf16 *)a.theta.shadow;
            e.grad_out = a.grad_out, e.flag = a.nonfinite, e.counter = nullptr, e.upd = upd;
            e.lr = a.lr, e.rho = a.rho, e.kappa = a.kappa;
            e.M = 512, e.N = 3136, e.pbase = P_W4, e.sbase = S_W4;
            tile<64, false, true>(c, LoadDense{a.dh1T, 512, n, a.n8}, LoadDense{a.act3[0][par], n, 3136, 3136}, e,
                                  0, (n + 63) / 64, mt * 128, nt * 64);
            break;
        }
        case J_B2D: {  // dY1 = relu'(x1) * transposed conv2(dY2), 4 input-parity classes
            const int tpc = counts_of(n).tpc;
            tile<64, false, true>(c, tconv_p(a.dY2, n, 10, 10, 9, 9, 64, tpc), weight_tp(tsh + S_W2, 64, 4, 32, tpc),
                                  epi_mask_p(a.dY1, a.act1[0], n, 10, 10, 32, tpc), 0, 4, j * 128, 0);
            break;
        }
        case J_B2W: {
            const int mt = j % 5, sp = j / 5;
            const int nch = (n * 81 + 63) / 64, kb0 = sp * a.kc2, kb1 = min(nch, kb0 + a.kc2);
            tile<64, true, true>(c, im2col(a.act1[0], n, 20, 20, 32, 4, 2, 9, 9), LoadDense{a.dY2, n * 81, 64, 64},
                                 EpiF32T{a.part2, 513, 64, 513, (size_t)64 * 513}, kb0, kb1, mt * 128, 0, sp,
                                 512, n * 81);
            break;
        }
        case J_B1W: {  // dW1^T[k][o] = sum_m P1[m][k] dY1[m][o] over uint8 frames; row 256 = ones
            const int mt = j % 3, sp = j / 3;
            const int nch = (n * 400 + 63) / 64, kb0 = sp * a.kc1, kb1 = min(nch, kb0 + a.kc1);
            tile<64, true, true>(c, frames(a.ring, a.records, map, nullptr, 0, n, REC_INTS, 0),
                                 LoadDense{a.dY1, n * 400, 32, 32}, EpiF32T{a.part1, 257, 32, 257, (size_t)32 * 257},
                                 kb0, kb1, mt * 128, 0, sp, 256, n * 400);
            break;
        }
        default: {  // RMSProp slices of the conv layers / fc1 bias / fc2
            OptArgs o{};
            o.p = a.theta.master, o.m = a.opt.m, o.v = a.opt.v;
            o.p2 = a.theta.master, o.m2 = a.opt.m, o.v2 = a.opt.v;
            o.shadow = (bf16 *)a.theta.shadow;
            o.part1 = a.part1, o.part2 = a.part2, o.part3 = a.part3, o.grad4 = nullptr;
            o.s1 = a.s1, o.s2 = a.s2, o.s3 = a.s3;
            o.dh1 = a.dh1, o.h1 = a.h1, o.td = a.td, o.act = a.act;
            o.n = n, o.A = a.A;
            o.lr = a.lr, o.rho = a.rho, o.kappa = a.kappa;
            o.flag = a.nonfinite, o.grad_out = a.grad_out;
            o.total = n_params(a.A);
            const int64_t lo = opt_lo(type) + (int64_t)j * PL_OPT_PER_JOB;
            const int64_t hi = min(opt_hi(type, a.A), lo + PL_OPT_PER_JOB);
#pragma unroll 1
            for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) opt_param(o, i, upd);
            break;
        }
    }
}

PQ_DEV void run_phase(const Ctx &c, const PhasePlan &P, int u) {
    const PLearnArgs &a = *c.a;
    int total = 0;
    for (int s = 0; s < P.nseg; ++s) {
        const Seg &g = P.seg[s];
        if (u + g.du < 0 || u + g.du >= a.n_updates) continue;
        total += g.end - g.begin;
    }
    for (int jid = blockIdx.x; jid < total; jid += gridDim.x) {
        int rem = jid;
        for (int s = 0; s < P.nseg; ++s) {
            const Seg &g = P.seg[s];
            if (u + g.du < 0 || u + g.du >= a.n_updates) continue;
            const int cnt = g.end - g.begin;
            if (rem < cnt) {
                run_job(c, g.type, g.grp, u + g.du, g.begin + rem);
                break;
            }
            rem -= cnt;
        }
    }
}

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_learn_persistent(const __grid_constant__ PLearnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[PL_STAGES];
    __shared__ uint32_t tmem_base_s;
    __shared__ int32_t table[TABLE_SAMPLES * 4];
    __shared__ int s_ubase;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) {
        for (int s = 0; s < PL_STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        s_ubase = *a.update_counter;
    }
    if ((threadIdx.x >> 5) == 0) tmem_alloc<64>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    TileRing R{smem, smem_u32(smem), bars, 0u, &tmem_base_s, table};
    const Ctx c{&a, &R, s_ubase};
    unsigned target = 0;
    int k = 0;  // phases run (trace row)
    auto phase = [&](const PhasePlan &P, int u) {
        run_phase(c, P, u);
        if (a.trace && threadIdx.x == 0) a.trace[((size_t)k * gridDim.x + blockIdx.x) * 2] = gtime();
        grid_barrier(a.bar, target);
        if (a.trace && threadIdx.x == 0) a.trace[((size_t)k * gridDim.x + blockIdx.x) * 2 + 1] = gtime();
        ++k;
    };
    {
        const Sched &S = a.sched[SCHED_PROLOGUE];
        for (int p = 0; p < S.nphases; ++p) phase(S.ph[p], 0);
    }
    for (int u = 0; u < a.n_updates; ++u) {
        const Sched &S = a.sched[u == a.n_updates - 1 ? SCHED_LAST : SCHED_STEADY];
        for (int p = 0; p < S.nphases; ++p) phase(S.ph[p], u);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.update_counter = s_ubase + a.n_updates;
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) tmem_dealloc<64>(tmem_base_s);
}

// ------------------------------------------------------------------ host side
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct PWS {
    bf16 *act1[2], *act2[2], *act3[2][2];
    float *fc1part[2][2];
    float *q, *h1, *dh1, *td;
    bf16 *dh1_bf, *dh1T;
    int32_t *act;
    bf16 *dY3, *dY2, *dY1;
    float *part1, *part2, *part3;
    unsigned *bar;
    size_t bytes;
};

static PWS carve_p(void *base, int N, int A) {
    PWS w;
    size_t off = 0;
    char *b = static_cast<char *>(base);
    auto take = [&](size_t bytes) -> void * {
        void *p = b ? b + off : nullptr;
        off += al(bytes);
        return p;
    };
    const int n8 = (N + 7) & ~7;
    for (int g = 0; g < 2; ++g) {
        w.act1[g] = (bf16 *)take((size_t)N * 400 * 32 * 2);
        w.act2[g] = (bf16 *)take((size_t)N * 81 * 64 * 2);
        for (int p = 0; p < 2; ++p) {
            w.act3[g][p] = (bf16 *)take((size_t)N * 3136 * 2);
            w.fc1part[g][p] = (float *)take((size_t)PL_FC1_SPLITS * N * 512 * 4);
        }
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
    w.part1 = (float *)take((size_t)MAX_SPLITS * 32 * 257 * 4);
    w.part2 = (float *)take((size_t)MAX_SPLITS * 64 * 513 * 4);
    w.part3 = (float *)take((size_t)MAX_SPLITS * 64 * 577 * 4);
    w.bar = (unsigned *)take(sizeof(unsigned));
    w.bytes = off;
    return w;
}

// split-K factor for `mtiles` M tiles of a contraction of `nch` 64-wide chunks given a
// CTA budget: chunks per split >= 2, splits <= MAX_SPLITS, table window for frames
static void choose_split(int nch, int mtiles, int budget, int kc_max, int *kc, int *splits) {
    int s = std::max(1, budget / mtiles);
    int k = std::max(2, (nch + s - 1) / s);
    k = std::max(k, (nch + MAX_SPLITS - 1) / MAX_SPLITS);
    k = std::min(k, kc_max);
    *kc = k;
    *splits = (nch + k - 1) / k;
}

struct PlanBuilder {
    Sched &S;
    int n, A, s1, s2, s3;
    PlanBuilder(Sched &s, int n_, int A_, int a, int b, int c) : S(s), n(n_), A(A_), s1(a), s2(b), s3(c) {}
    int count(int type) const { return njobs(type, n, A, s1, s2, s3); }
    void add(int p, int type, int grp, int du, int begin = 0, int end = -1) {
        if (end < 0) end = count(type);
        if (end <= begin) return;
        PhasePlan &P = S.ph[p];
        P.seg[P.nseg++] = Seg{(int16_t)type, (int8_t)grp, (int8_t)du, begin, end};
        S.nphases = std::max(S.nphases, p + 1);
    }
    int load(int p) const {
        int t = 0;
        for (int s = 0; s < S.ph[p].nseg; ++s) t += S.ph[p].seg[s].end - S.ph[p].seg[s].begin;
        return t;
    }
};

static void build_plans(PLearnArgs &a, int G) {
    const int n = a.n, A = a.A;
    const Counts cn = counts_of(n);
    memset(a.sched, 0, sizeof(a.sched));
    choose_split((n * 400 + 63) / 64, 3, G, (TABLE_SAMPLES - 2) * 400 / 64, &a.kc1, &a.s1);
    choose_split((n * 81 + 63) / 64, 5, std::max(5, G - 4 * cn.tpc), 1 << 20, &a.kc2, &a.s2);
    choose_split((n * 49 + 63) / 64, 5, std::max(5, G - cn.t2), 1 << 20, &a.kc3, &a.s3);
    {  // prologue: the target forward of the launch's first step
        PlanBuilder b(a.sched[SCHED_PROLOGUE], n, A, a.s1, a.s2, a.s3);
        b.add(0, J_F1, 1, 0);
        b.add(1, J_F2, 1, 0);
        b.add(2, J_F3, 1, 0);
        b.add(3, J_F4, 1, 0);
    }
    for (int last = 0; last < 2; ++last) {
        PlanBuilder b(a.sched[last ? SCHED_LAST : SCHED_STEADY], n, A, a.s1, a.s2, a.s3);
        b.add(0, J_F1, 0, 0);
        b.add(1, J_F2, 0, 0);
        b.add(2, J_F3, 0, 0);
        b.add(3, J_F4, 0, 0);
        b.add(4, J_HEAD, 0, 0);
        b.add(5, J_B4D, 0, 0);
        b.add(5, J_OPT_FC2, 0, 0);
        b.add(6, J_B3D, 0, 0);
        b.add(6, J_B3W, 0, 0);
        b.add(7, J_B2D, 0, 0);
        b.add(7, J_B2W, 0, 0);
        b.add(8, J_B1W, 0, 0);
        b.add(9, J_OPT_C1, 0, 0);
        b.add(9, J_OPT_C2, 0, 0);
        b.add(9, J_OPT_C3, 0, 0);
        if (!last) {  // target forward of the next step
            b.add(1, J_F1, 1, +1);
            b.add(2, J_F2, 1, +1);
            b.add(3, J_F3, 1, +1);
            b.add(4, J_F4, 1, +1);
        }
    }
    // fc1 weight gradient + RMSProp tiles (196) into the spare CTAs of the phases where
    // they may run: 6-9 of their own step, 0-2 of the next (du = -1 there).  The split
    // is decided for a steady step; the last step of a launch runs the previous step's
    // leftovers in 0-2 as usual and all of its own tiles in 6-9.
    PlanBuilder st(a.sched[SCHED_STEADY], n, A, a.s1, a.s2, a.s3);
    PlanBuilder ls(a.sched[SCHED_LAST], n, A, a.s1, a.s2, a.s3);
    st.S.nphases = ls.S.nphases = 10;
    const int total = st.count(J_B4W);
    const int own[4] = {6, 7, 8, 9}, nxt[3] = {0, 1, 2};
    int next = 0;
    for (int p : own) {
        const int take = std::min(total - next, std::max(0, G - st.load(p)));
        if (take > 0) st.add(p, J_B4W, 0, 0, next, next + take);
        next += std::max(0, take);
    }
    for (int p : nxt) {
        const int take = std::min(total - next, std::max(0, G - st.load(p)));
        if (take > 0) {
            st.add(p, J_B4W, 0, -1, next, next + take);
            ls.add(p, J_B4W, 0, -1, next, next + take);
        }
        next += std::max(0, take);
    }
    if (next < total) st.add(9, J_B4W, 0, 0, next, total);
    next = 0;
    for (int p : own) {
        int take = std::min(total - next, std::max(0, G - ls.load(p)));
        if (p == 9) take = total - next;
        if (take > 0) ls.add(p, J_B4W, 0, 0, next, next + take);
        next += std::max(0, take);
    }
}

static int g_learn_ctas = 0;  // 0 = all SMs minus the acting reserve
static unsigned long long *g_trace = nullptr;

}  // namespace pq

using namespace pq;

extern "C" {

size_t pq_plearn_workspace_bytes(int max_batch, int actions) {
    return carve_p(nullptr, max_batch, actions).bytes;
}

int pq_plearn_set_ctas(int ctas) {
    g_learn_ctas = ctas;
    return 0;
}

// the GEMM timeline probes of this translation unit's tiles (see pq_timeline)
int pq_plearn_timeline(int on, unsigned long long *out, int *count) {
    if (out) {
        static Timeline h;
        PQ_CUDA_TRY(cudaMemcpyFromSymbol(&h, g_tl, sizeof(Timeline)));
        *count = h.n < 256 ? h.n : 256;
        memcpy(out, h.t, sizeof(h.t));
    }
    Timeline z{};
    z.on = on;
    PQ_CUDA_TRY(cudaMemcpyToSymbol(g_tl, &z, sizeof(int) * 2));
    return 0;
}

int pq_plearn_trace(unsigned long long *device_buf) {
    g_trace = device_buf;
    return 0;
}

int pq_learn_run(const pq_learn_args *la, int n_updates, void *stream) {
    const int n = la->n;
    if (n < 1 || n > la->max_batch) return set_err("batch size out of range for the workspace");
    if (la->actions < 1 || la->actions > MAX_ACTIONS) return set_err("actions must be in [1, 32]");
    if (n_updates < 1) return set_err("n_updates must be >= 1");
    if (la->ext_targets || la->idx || !la->idx_base || !la->update_counter)
        return set_err("persistent learner: needs the epoch index table + update counter, no external targets");
    if (la->theta_out.master != la->theta.master || la->opt_out.m != la->opt.m)
        return set_err("persistent learner: updates theta / opt in place");
    cudaStream_t st = (cudaStream_t)stream;
    static int sms = 0;
    static bool configured = false;
    if (!configured) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_learn_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, PL_SMEM));
        configured = true;
    }
    const int G = g_learn_ctas > 0 ? std::min(g_learn_ctas, sms) : std::max(1, sms - 20);
    PWS w = carve_p(la->ws, la->max_batch, la->actions);
    PLearnArgs a;
    memset(&a, 0, sizeof(a));
    a.theta = la->theta, a.target = la->target, a.opt = la->opt;
    a.ring = la->ring, a.records = la->records, a.idx_base = la->idx_base;
    a.update_counter = la->update_counter;
    a.n = n, a.A = la->actions, a.n8 = (n + 7) & ~7, a.n_updates = n_updates;
    a.gamma = la->gamma, a.lr = la->lr, a.rho = la->rho, a.kappa = la->kappa;
    a.nonfinite = la->nonfinite, a.grad_out = la->grad_out, a.q_out = la->q_out, a.td_out = la->td_out;
    for (int g = 0; g < 2; ++g) {
        a.act1[g] = w.act1[g], a.act2[g] = w.act2[g];
        for (int p = 0; p < 2; ++p) a.act3[g][p] = w.act3[g][p], a.fc1part[g][p] = w.fc1part[g][p];
    }
    a.q = w.q, a.h1 = w.h1, a.dh1 = w.dh1, a.td = w.td, a.dh1_bf = w.dh1_bf, a.dh1T = w.dh1T, a.act = w.act;
    a.dY3 = w.dY3, a.dY2 = w.dY2, a.dY1 = w.dY1;
    a.part1 = w.part1, a.part2 = w.part2, a.part3 = w.part3;
    a.bar = w.bar;
    a.trace = g_trace;
    build_plans(a, G);
    PQ_CUDA_TRY(cudaMemsetAsync(w.bar, 0, sizeof(unsigned), st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = PL_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_err(cudaLaunchKernelEx(&cfg, k_learn_persistent, a), "persistent learner");
}

}  // extern "C"
