// Persistent DQN learner: many learner steps (agent.train_minibatch, agent.py:84-105)
// in ONE launch of one 256-thread CTA per SM, every GEMM operand moved by TMA.
//
// A batch-32 step is ~2 GFLOP spread over ten dependent GEMM-shaped stages.  As separate
// launches with per-thread cp.async gathers it is a chain of launch / drain latencies and
// of instruction-bound operand address generation (IPC ~1, ~235 SASS instructions per
// warp per K-chunk; profiles/r1_v9_summary.md).  Here:
//
//  * every CTA keeps its TMEM accumulator, operand ring and mbarriers for the whole
//    launch; the stages of a step are PHASES separated by a grid barrier; each phase is
//    a list of jobs (GEMM tiles, head samples, optimizer slices, frame gathers) dealt
//    round-robin to the CTAs;
//  * every GEMM operand is a dense row-major matrix fetched by cp.async.bulk.tensor
//    (128B-swizzled 64x64 boxes, one thread issues a K-chunk's 2-3 boxes): the im2col
//    matrices of conv2 / conv3 and of the two transposed convolutions are SCATTERED by
//    the epilogue that produces the activation / gradient (each element lands in the
//    <= 9 patch rows it belongs to), and the conv1 patch matrix of the sampled uint8
//    frame stacks is built by a gather job ahead of time (the epoch's indices are known);
//    bias gradients ride on a constant ones column of those matrices;
//  * the mainloop is warp-specialised: thread 0 produces (empty -> expect_tx -> TMA),
//    thread 32 issues tcgen05.mma and commits to the slot's empty barrier and to the
//    accumulator barrier, all 8 warps run the epilogue from TMEM;
//  * work off the critical chain rides in the idle CTAs of other phases: the
//    target-network forward of step u+1 (theta-minus and the indices are fixed for the
//    launch), the frame gathers of steps u+1 / u+2, and the fc1 weight gradient + fused
//    RMSProp (196 tiles, the HBM-heavy stage) spread over phases 6-9 of step u and 0-2
//    of step u+1 (act3 double-buffered by step parity).
//
// Phase plan of step u (critical job first, fillers after):
//   P0 F1 online conv1            | fc1 wgrad+RMS (u-1)
//   P1 F2 online conv2            | F1 target (u+1) | fc1 wgrad+RMS (u-1)
//   P2 F3 online conv3            | F2 target (u+1) | fc1 wgrad+RMS (u-1)
//   P3 F4 online fc1 (split-K)    | F3 target (u+1)
//   P4 head (fc2, TD target, delta, fc2 back-prop) | F4 target (u+1)
//   P5 fc1 dgrad                  | fc2 / fc1-bias RMSProp | frame gather target (u+2)
//   P6 conv3 dgrad, conv3 wgrad   | fc1 wgrad+RMS
//   P7 conv2 dgrad, conv2 wgrad   | fc1 wgrad+RMS
//   P8 conv1 wgrad                | fc1 wgrad+RMS
//   P9 conv1/2/3 RMSProp          | frame gather online (u+1) | fc1 wgrad+RMS
// The arithmetic of each stage is the one-shot path's (same K order, epilogues, head and
// optimizer functions); the two agree to fp32 split-K summation order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "../../include/paraq_b200.h"
#include "learn_parts.cuh"

namespace pq {
int set_err(const char *msg);
int cuda_err(cudaError_t e, const char *where);
#define PQ_CUDA_TRY(expr)                  \
    do {                                   \
        int _rc = cuda_err((expr), #expr); \
        if (_rc) return _rc;               \
    } while (0)

constexpr int PL_STAGES = 8;
constexpr int PL_SLOT = 24 * 1024;  // A: two 8 KB boxes, B: one 8 KB box
constexpr int PL_B_OFF = 16 * 1024;
constexpr int PL_SMEM = PL_STAGES * PL_SLOT + 1024;
constexpr int PL_BOX = 8192;        // one 64 x 64 bf16 box, 128B-swizzled
constexpr int PL_FC1_KC = 3;        // fc1 forward: 49 K-chunks in 17 splits
constexpr int PL_FC1_SPLITS = (49 + PL_FC1_KC - 1) / PL_FC1_KC;
constexpr int PL_OPT_PER_JOB = 256;  // parameters per optimizer job (one per thread)
// padded widths of the patch matrices (bf16 elements; 16-byte row strides)
constexpr int P1_LD = 320, P2_LD = 576;

enum Job : int16_t {
    J_F1, J_F2, J_F3, J_F4, J_HEAD, J_B4D, J_OPT_FC2, J_B3D, J_B3W, J_B4W, J_B2D, J_B2W,
    J_OPT_C3, J_B1W, J_OPT_C2, J_OPT_C1, J_G1, J_COUNT
};

// tensor maps
enum Map {
    M_W1 = 0, M_W2 = 2, M_W3 = 4, M_W4 = 6,  // [g]
    M_ACT3 = 8,                              // [g][par]
    M_P1 = 12,                               // [g][par]
    M_P2 = 16, M_ACT2I = 18,                 // [g]  ACT2I: im2col map of act2, 128 pixels
    M_ACT2W = 20,                            // im2col map of act2 (online), 64 pixels (wgrad)
    M_DY3I, M_DY2I, M_ONES, M_DH1, M_DH1T, M_DY3, M_DY2, M_DY1, M_W3V, M_W2V, M_COUNT
};

struct Seg {
    int16_t type;
    int8_t grp;     // 0 online, 1 target (forward / gather jobs)
    int8_t du;      // step offset of the job relative to the running step
    int16_t filler; // off the step's critical chain: dealt to the CTAs without a critical job
    int16_t pad;
    int32_t begin, end;
};
constexpr int PL_MAX_PHASES = 12, PL_MAX_SEGS = 8;
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
    CUtensorMap maps[M_COUNT];
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
    bf16 *wsb;  // base of the workspace (lowest buffer)
    bf16 *act1, *act2[2], *act3[2][2];
    bf16 *ones;  // [64][64], column 0 = 1: the bias-gradient atom of the conv3 wgrad
    bf16 *P1[2][2], *P2[2];
    float *fc1part[2][2];
    float *q, *h1, *dh1, *td;
    bf16 *dh1_bf, *dh1T;
    int32_t *act;
    bf16 *dY3, *dY2, *dY1;
    float *part1, *part2, *part3;
    int s1, s2, s3, kc1, kc2, kc3;
    unsigned *bar;
    unsigned long long *trace;  // optional [phases run][gridDim][4]: jobs done, barrier passed, last job type, its ns
    Sched sched[3];
};

// ------------------------------------------------------------------ job counts
struct Counts {
    int t1, t2, t3, nt64, mt128, tpc;
};
__host__ __device__ inline Counts counts_of(int n) {
    Counts c;
    c.t1 = (n * 400 + 127) / 128;
    c.t2 = (n * 81 + 127) / 128;
    c.t3 = (n * 49 + 127) / 128;
    c.nt64 = (n + 63) / 64;
    c.mt128 = (n + 127) / 128;
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
        case J_F4: return 4 * c.nt64 * PL_FC1_SPLITS;
        case J_HEAD: return n;
        case J_B4D: return c.mt128 * 49;
        case J_B3D: return c.t2;
        case J_B3W: return 5 * s3;
        case J_B4W: return 4 * 49;
        case J_B2D: return 4 * c.tpc;
        case J_B2W: return 5 * s2;
        case J_B1W: return 3 * s1;
        case J_G1: return 4 * n;  // quarter samples (100 patch rows each)
        default: return (int)((opt_hi(type, A) - opt_lo(type) + PL_OPT_PER_JOB - 1) / PL_OPT_PER_JOB);
    }
}

// ------------------------------------------------------------------ grid barrier
// Monotonic arrival counter (zeroed before the launch); the k-th barrier completes when
// it reaches k * gridDim.x.  gpu-scope fences on both sides (they also invalidate the
// SM's L1 so later plain loads see other CTAs' writes).
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

template <class EP, class = void>
struct is_scatter {
    static constexpr bool value = false;
};
template <class EP>
struct is_scatter<EP, decltype((void)EP::NDEST)> {
    static constexpr bool value = true;
};

// ------------------------------------------------------------------ TMA GEMM tile
// One operand of a K-chunk: `boxes` 64x64 boxes of a tiled tensor map, or an im2col
// load of an NHWC activation / gradient (hardware patch gather, zero padding):
//   K2:  K-major rows r0 + 64b, columns 64 kb          (row-major [MN][K] matrix)
//   M2:  MN-major columns r0 + 64b, rows 64 kb         (row-major [K][MN] matrix)
//   W3V: conv3 weight as [c][(kh,kw)][o]: tap kb      (MN-major B of the conv3 dgrad)
//   W2V: conv2 weight as [c][kw][kh][o]: tap of the parity class (conv2 dgrad)
//   IF3: conv3 forward patches of act2 (9x9x64 -> 7x7), 128 output pixels from r0, tap kb
//   IT3: conv3 transposed-conv window of dY3 (7x7x64 -> 9x9, padding 2), tap kb
//   IT2: conv2 parity-class transposed-conv window of dY2 (9x9x64 -> 10x10, padding 1)
//   IW3: conv3 patches of act2 as the MN-major A of the conv3 weight gradient: K-chunk =
//        64 output pixels from 64 kb, MN atoms = taps 2 mt, 2 mt + 1; tap 9 = the ones
//        tile (bias gradient: column 0 = 1)
//   IF1: conv1 forward over the space-to-depth frame stacks (21x21 pixels x 16 sub-pixels
//        per frame): 2x2 taps, 128 output pixels from r0, channels from cls (16 g)
//   IW1: the same patches as the MN-major A of the conv1 weight gradient (64 pixels per
//        K-chunk, taps 2 mt, 2 mt + 1; tap 4 = the ones tile, tap 5 = zeros)
enum { OP_K2, OP_M2, OP_W3V, OP_W2V, OP_IF3, OP_IT3, OP_IT2, OP_IW3, OP_IF1, OP_IW1 };
struct TmaOp {
    const CUtensorMap *map;
    int kind, boxes, r0, cls, n;
    const CUtensorMap *aux;  // IW3: the ones tile
    PQ_DEV void issue(uint32_t dst, uint64_t *bar, int kb, int lane) const {
        if (lane != 0) return;
        switch (kind) {
            case OP_K2:
                for (int b = 0; b < boxes; ++b) tma_load_2d(dst + b * PL_BOX, map, bar, kb * 64, r0 + 64 * b);
                break;
            case OP_M2:
                for (int b = 0; b < boxes; ++b) tma_load_2d(dst + b * PL_BOX, map, bar, r0 + 64 * b, kb * 64);
                break;
            case OP_W3V:
                tma_load_3d(dst, map, bar, 0, kb, 0);
                break;
            case OP_W2V: {
                const int kh = (cls >> 1) + 2 * (kb >> 1), kw = (cls & 1) + 2 * (kb & 1);
                tma_load_4d(dst, map, bar, 0, kw, kh, 0);
                break;
            }
            case OP_IF3: {  // output pixel r0 = (b, oy, ox) of 7x7; input base (ox, oy), tap offset
                const int b = r0 / 49, q = r0 - b * 49, oy = q / 7, ox = q - oy * 7;
                const int kh = kb / 3, kw = kb - kh * 3;
                tma_im2col_4d(dst, map, bar, 0, ox, oy, b, (uint16_t)kw, (uint16_t)kh);
                break;
            }
            case OP_IT3: {  // input pixel r0 = (b, iy, ix) of 9x9 reads dY3[iy - kh][ix - kw]
                const int b = r0 / 81, q = r0 - b * 81, iy = q / 9, ix = q - iy * 9;
                const int kh = kb / 3, kw = kb - kh * 3;
                tma_im2col_4d(dst, map, bar, 0, ix - 2, iy - 2, b, (uint16_t)(2 - kw), (uint16_t)(2 - kh));
                break;
            }
            case OP_IT2: {  // class-local row r0 = (b, iy', ix') of 10x10 reads dY2[iy' - ty][ix' - tx]
                const int b = r0 / 100, q = r0 - b * 100, iy = q / 10, ix = q - iy * 10;
                const int ty = kb >> 1, tx = kb & 1;
                tma_im2col_4d(dst, map, bar, 0, ix - 1, iy - 1, b, (uint16_t)(1 - tx), (uint16_t)(1 - ty));
                break;
            }
            case OP_IF1: {
                const int b = r0 / 400, q = r0 - b * 400, oy = q / 20, ox = q - oy * 20;
                tma_im2col_4d(dst, map, bar, cls, ox, oy, b, (uint16_t)(kb & 1), (uint16_t)(kb >> 1));
                break;
            }
            case OP_IW1: {
                const int p0 = kb * 64, b = p0 / 400, q = p0 - b * 400, oy = q / 20, ox = q - oy * 20;
                for (int atom = 0; atom < 2; ++atom) {
                    const int t = 2 * (r0 >> 7) + atom;
                    if (t < 4)
                        tma_im2col_4d(dst + atom * PL_BOX, map, bar, 0, ox, oy, b, (uint16_t)(t & 1), (uint16_t)(t >> 1));
                    else  // ones tile (bias row), then a fully out-of-bounds box = zeros
                        tma_load_2d(dst + atom * PL_BOX, aux, bar, t == 4 ? 0 : 64, 0);
                }
                break;
            }
            default: {  // OP_IW3
                const int p0 = kb * 64, b = p0 / 49, q = p0 - b * 49, oy = q / 7, ox = q - oy * 7;
                for (int atom = 0; atom < 2; ++atom) {
                    const int t = 2 * (r0 >> 7) + atom;
                    if (t < 9) {
                        const int kh = t / 3, kw = t - kh * 3;
                        tma_im2col_4d(dst + atom * PL_BOX, map, bar, 0, ox, oy, b, (uint16_t)kw, (uint16_t)kh);
                    } else {
                        tma_load_2d(dst + atom * PL_BOX, aux, bar, 0, 0);
                    }
                }
                break;
            }
        }
    }
};

// latency probe of CTA 0's tiles (pq_plearn_timeline): thread-0 timestamps in shared
// memory, copied out at the end of the tile
__shared__ unsigned long long s_tl[8];
#define PL_PROBE(i)                                                                \
    do {                                                                           \
        if (g_tl.on && blockIdx.x == 0 && threadIdx.x == 0) s_tl[i] = gtime(); \
    } while (0)

struct Pipe {
    uint8_t *smem;
    uint32_t smem_s;
    uint64_t *full, *empty, *acc;
    uint32_t seq, tiles;
    const uint32_t *tmem_s;
};

// 128 x BN tile over K-chunks [kb0, kb1): thread 0 streams the operand boxes into the
// ring (waiting on each slot's empty barrier), thread 32 issues 4 x tcgen05.mma per
// chunk and commits the slot back, then the accumulator; all threads run the epilogue.
template <int BN, bool AMN, bool BMN, class EP>
PQ_DEV void tma_tile(const TmaOp &A, const TmaOp &B, const EP &ep, int kb0, int kb1, int m0, int n0,
                     int split, Pipe &P) {
    constexpr uint32_t IDESC = idesc_bf16(BN, AMN, BMN);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = kb1 > kb0 ? kb1 - kb0 : 0;
    const uint32_t seq0 = P.seq;
    const uint32_t tmem = *P.tmem_s;
    PL_PROBE(0);
    if (g_tl.on && blockIdx.x == 0 && tid == 0) s_tl[2] = s_tl[3] = 0;
    if (warp == 0) {  // producer warp: lane 0 arms the slot, every lane may gather
        const uint32_t bytes = (uint32_t)(A.boxes + B.boxes) * PL_BOX;
        for (int i = 0; i < nk; ++i) {
            const uint32_t q = seq0 + i, s = q % PL_STAGES;
            if (lane == 0) {
                if (q >= PL_STAGES) mbar_wait(&P.empty[s], ((q / PL_STAGES) - 1) & 1);
                mbar_expect_tx(&P.full[s], bytes);
            }
            const uint32_t dst = P.smem_s + s * PL_SLOT;
            A.issue(dst, &P.full[s], kb0 + i, lane);
            B.issue(dst + PL_B_OFF, &P.full[s], kb0 + i, lane);
        }
    } else if (tid == 32) {
        for (int i = 0; i < nk; ++i) {
            const uint32_t q = seq0 + i, s = q % PL_STAGES;
            mbar_wait(&P.full[s], (q / PL_STAGES) & 1);
            tc_fence_after();
            const uint32_t a_addr = P.smem_s + s * PL_SLOT, b_addr = a_addr + PL_B_OFF;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t ad = AMN ? desc_sw128(a_addr + j * 2048, 8192) : desc_sw128(a_addr + j * 32, 0);
                const uint64_t bd = BMN ? desc_sw128(b_addr + j * 2048, 8192) : desc_sw128(b_addr + j * 32, 0);
                umma_bf16(tmem, ad, bd, IDESC, (i > 0 || j > 0) ? 1u : 0u);
            }
            umma_commit(&P.empty[s]);
        }
        umma_commit(P.acc);
    }
    mbar_wait(P.acc, P.tiles & 1);
    PL_PROBE(1);
    __syncwarp();
    tc_fence_after();
    P.seq = seq0 + nk;
    P.tiles += 1;

    const int wq = warp & 3, half = warp >> 2;
    const int row = m0 + wq * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    constexpr int CW = BN >= 64 ? BN / 2 : BN;
    if constexpr (is_scatter<EP>::value) {
        // bf16 results staged in the idle ring, then written as whole 16-byte chunks of
        // each destination row segment (consecutive lanes -> consecutive chunks)
        constexpr int TS = BN + 8;  // padded row stride (elements): conflict-free 16B stores
        bf16 *tile = reinterpret_cast<bf16 *>(P.smem);
        const int cbeg = BN >= 64 ? half * CW : 0;
        if ((BN >= 64 || half == 0) && cbeg < EP::ROW_CHUNKS * 8) {
            for (int c0 = cbeg; c0 < cbeg + CW && c0 < EP::ROW_CHUNKS * 8; c0 += 32) {
                float v[32];
                if (nk > 0) {
                    tmem_ld32(trow + c0, v);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
                uint4 o[4];
                ep.compute(row, n0 + c0, v, o);
                uint4 *d = reinterpret_cast<uint4 *>(tile + (wq * 32 + lane) * TS + c0);
#pragma unroll
                for (int q = 0; q < 4; ++q) d[q] = o[q];
            }
        }
        PL_PROBE(2);
        // destination offsets of every (row, segment) once, then whole-chunk copies
        int32_t *dtab = reinterpret_cast<int32_t *>(P.smem + 128 * TS * 2);
        if (tid < 128) {
#pragma unroll 1
            for (int k = 0; k < EP::NDEST; ++k) {
                const bf16 *d = ep.dest(m0 + tid, n0, k);
                dtab[k * 128 + tid] = d ? (int32_t)(d - ep.wsb) : -1;
            }
        }
        __syncthreads();
        PL_PROBE(3);
        constexpr int CH = EP::ROW_CHUNKS;
        bf16 *base = ep.wsb;
#pragma unroll 1
        for (int e = tid; e < EP::NDEST * 128 * CH; e += GEMM_THREADS) {
            const int ch = e % CH, rk = e / CH;  // rk = k * 128 + r
            const int off = dtab[rk];
            if (off >= 0)
                *reinterpret_cast<uint4 *>(base + (size_t)(uint32_t)off + ch * 8) =
                    *reinterpret_cast<const uint4 *>(tile + (rk & 127) * TS + ch * 8);
        }
    } else if constexpr (is_staged<EP>::value) {
        static_assert(128 * (BN + 1) * 4 <= PL_STAGES * PL_SLOT, "staging tile");
        float *tile = reinterpret_cast<float *>(P.smem);
        if (BN >= 64 || half == 0) {
            const int cbeg = BN >= 64 ? half * CW : 0;
            for (int c0 = cbeg; c0 < cbeg + CW; c0 += 32) {
                float v[32];
                if (nk > 0) {
                    tmem_ld32(trow + c0, v);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) tile[(wq * 32 + lane) * (BN + 1) + c0 + e] = v[e];
            }
        }
        __syncthreads();
        ep.template apply_tile<BN>(tile, BN + 1, m0, n0);
    } else if (BN >= 64 || half == 0) {
        const int cbeg = BN >= 64 ? half * CW : 0;
#pragma unroll 1
        for (int c0 = cbeg; c0 < cbeg + CW; c0 += 32) {
            float v[32];
            if (nk > 0) {
                tmem_ld32(trow + c0, v);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.f;
            }
            ep.apply(row, n0 + c0, v, 32, split);
        }
    }
    PL_PROBE(4);
    tc_fence_before();
    __syncthreads();
    if (g_tl.on && blockIdx.x == 0 && threadIdx.x == 0) {
        s_tl[5] = gtime();
        const int slot = atomicAdd(&g_tl.n, 1);
        if (slot < 256) {
            for (int k = 0; k < 6; ++k) g_tl.t[slot][k] = s_tl[k];
            g_tl.t[slot][6] = (unsigned long long)nk;
            g_tl.t[slot][7] = (unsigned long long)BN;
        }
    }
}

// ------------------------------------------------------------------ scatter epilogues
PQ_DEV void relu_pack(const float *v, const float *bias, float scale, uint4 (&o)[4]) {
    float y[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
        const float t = v[e] * scale + bias[e];
        y[e] = t > 0.f ? t : 0.f;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
        o[c] = make_uint4(pack_bf16(y[8 * c], y[8 * c + 1]), pack_bf16(y[8 * c + 2], y[8 * c + 3]),
                          pack_bf16(y[8 * c + 4], y[8 * c + 5]), pack_bf16(y[8 * c + 6], y[8 * c + 7]));
}
PQ_DEV void store64(bf16 *dst, const uint4 (&o)[4]) {
    uint4 *d = reinterpret_cast<uint4 *>(dst);
#pragma unroll
    for (int c = 0; c < 4; ++c) d[c] = o[c];
}
// masked (relu') copy of 32 values: mask = forward activation at the same place
PQ_DEV void mask_pack(const float *v, const bf16 *mask, uint4 (&o)[4]) {
    uint4 mk[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) mk[c] = __ldcg(reinterpret_cast<const uint4 *>(mask) + c);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t mw[4] = {mk[c].x, mk[c].y, mk[c].z, mk[c].w};
        uint32_t r[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float a = bf16_lo(mw[e]) > 0.f ? v[8 * c + 2 * e] : 0.f;
            const float b = bf16_hi(mw[e]) > 0.f ? v[8 * c + 2 * e + 1] : 0.f;
            r[e] = pack_bf16(a, b);
        }
        o[c] = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// Scatter epilogues: compute() turns 32 accumulator columns of a row into bf16
// (bias + ReLU, or the relu' mask), dest(m, n0, k) names the k-th row segment that
// receives the staged row (nullptr = none); ROW_CHUNKS 16-byte chunks per segment.

// conv1: rows (b, oy, ox) of 20x20, 32 channels -> act1 (online, the relu' mask of the
// conv2 dgrad) and the conv2 patch rows (b, oy2, ox2) col (kh, kw, c), oy = 2 oy2 + kh
struct EpiConv1 {
    static constexpr int NDEST = 5, ROW_CHUNKS = 4;
    bf16 *wsb;  // workspace base: destinations are int32 element offsets from it
    bf16 *act1, *P2;
    const float *bias;
    int n;
    float scale;
    PQ_DEV void compute(int, int n0, const float *v, uint4 (&o)[4]) const {
        float bv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) bv[e] = __ldcg(bias + n0 + e);
        relu_pack(v, bv, scale, o);
    }
    PQ_DEV bf16 *dest(int m, int, int k) const {
        if (m >= n * 400) return nullptr;
        if (k == 0) return act1 ? act1 + (size_t)m * 32 : nullptr;
        const int b = m / 400, p = m - b * 400, oy = p / 20, ox = p - oy * 20;
        const int kh = (oy & 1) + 2 * ((k - 1) >> 1), kw = (ox & 1) + 2 * ((k - 1) & 1);
        const int oy2 = (oy - kh) >> 1, ox2 = (ox - kw) >> 1;
        if (oy2 < 0 || oy2 > 8 || ox2 < 0 || ox2 > 8) return nullptr;
        return P2 + (size_t)(b * 81 + oy2 * 9 + ox2) * P2_LD + (kh * 4 + kw) * 32;
    }
};

// conv2: rows (b, oy, ox) of 9x9, 64 channels -> act2 (gathered by conv3's TMA and
// the relu' mask of the conv3 dgrad)
struct EpiConv2 {
    static constexpr int NDEST = 1, ROW_CHUNKS = 8;
    bf16 *wsb;  // workspace base: destinations are int32 element offsets from it
    bf16 *act2;
    const float *bias;
    int n;
    PQ_DEV void compute(int, int n0, const float *v, uint4 (&o)[4]) const {
        float bv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) bv[e] = __ldcg(bias + n0 + e);
        relu_pack(v, bv, 1.0f, o);
    }
    PQ_DEV bf16 *dest(int m, int, int) const { return m < n * 81 ? act2 + (size_t)m * 64 : nullptr; }
};

// conv3 forward: rows (b, p) -> act3 [b][p][64] (dense)
struct EpiConv3 {
    static constexpr int NDEST = 1, ROW_CHUNKS = 8;
    bf16 *wsb;  // workspace base: destinations are int32 element offsets from it
    bf16 *act3;
    const float *bias;
    int n;
    PQ_DEV void compute(int, int n0, const float *v, uint4 (&o)[4]) const {
        float bv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) bv[e] = __ldcg(bias + n0 + e);
        relu_pack(v, bv, 1.0f, o);
    }
    PQ_DEV bf16 *dest(int m, int, int) const { return m < n * 49 ? act3 + (size_t)m * 64 : nullptr; }
};

// fc1 data gradient (rows = samples, the 64 cols of a tile = the 64 channels of one
// conv3 output pixel p): dY3 = acc * relu'(act3)
struct EpiB4D {
    static constexpr int NDEST = 1, ROW_CHUNKS = 8;
    bf16 *wsb;  // workspace base: destinations are int32 element offsets from it
    bf16 *dY3;
    const bf16 *act3;
    int n;
    PQ_DEV void compute(int m, int n0, const float *v, uint4 (&o)[4]) const {
        if (m < n) {
            mask_pack(v, act3 + (size_t)m * 3136 + n0, o);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = make_uint4(0, 0, 0, 0);
        }
    }
    PQ_DEV bf16 *dest(int m, int n0, int) const { return m < n ? dY3 + (size_t)m * 3136 + n0 : nullptr; }
};

// conv3 data gradient (rows (b, iy, ix) of 9x9): dY2 = acc * relu'(act2)
struct EpiB3D {
    static constexpr int NDEST = 1, ROW_CHUNKS = 8;
    bf16 *wsb;  // workspace base: destinations are int32 element offsets from it
    bf16 *dY2;
    const bf16 *act2;
    int n;
    PQ_DEV void compute(int m, int n0, const float *v, uint4 (&o)[4]) const {
        if (m < n * 81) {
            mask_pack(v, act2 + (size_t)m * 64 + n0, o);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = make_uint4(0, 0, 0, 0);
        }
    }
    PQ_DEV bf16 *dest(int m, int, int) const { return m < n * 81 ? dY2 + (size_t)m * 64 : nullptr; }
};

// conv2 data gradient per parity class (rows class-major, (b, iy', ix') of 10x10, 32
// channels): dY1 = acc * relu'(act1) at NHWC position (2 iy' + py, 2 ix' + px)
struct EpiB2D {
    static constexpr int NDEST = 1, ROW_CHUNKS = 4;
    bf16 *wsb;  // workspace base: destinations are int32 element offsets from it
    bf16 *dY1;
    const bf16 *act1;
    int n, tpc;
    PQ_DEV int64_t pos(int m) const {
        const int cls = m / (tpc * 128), loc = m - cls * tpc * 128;
        if (loc >= n * 100) return -1;
        const int b = loc / 100, r = loc - b * 100, ry = r / 10, rx = r - ry * 10;
        const int iy = 2 * ry + (cls >> 1), ix = 2 * rx + (cls & 1);
        return ((int64_t)(b * 20 + iy) * 20 + ix) * 32;
    }
    PQ_DEV void compute(int m, int n0, const float *v, uint4 (&o)[4]) const {
        const int64_t q = pos(m);
        if (q >= 0) {
            mask_pack(v, act1 + q + n0, o);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) o[c] = make_uint4(0, 0, 0, 0);
        }
    }
    PQ_DEV bf16 *dest(int m, int, int) const {
        const int64_t q = pos(m);
        return q >= 0 ? dY1 + q : nullptr;
    }
};

// ------------------------------------------------------------------ jobs
struct Ctx {
    const PLearnArgs *a;
    Pipe *P;
    int u_base;
    int k;  // phases run (trace row)
};

PQ_DEV TmaOp op(const PLearnArgs &a, int map, int kind, int boxes, int r0, int cls = 0) {
    return TmaOp{&a.maps[map], kind, boxes, r0, cls, a.n, &a.maps[M_ONES]};
}

// conv1 patch rows of sample b (g = 0: state frames f0..f3, 1: next state f1..f4):
// P1[(b, oy, ox)][k'(c, kh, kw)] = frame_c[4 oy + kh][4 ox + kw] (permuted K; 0..255 in bf16;
// the 1/255 input scale is applied in the conv1 epilogue); slot -1 = masked zero frame.
// The 4 frames are staged in the (idle) operand ring with coalesced 16-byte loads, all
// in flight together; the patch rows leave as consecutive 16-byte chunks.
PQ_DEV void gather_patches(const PLearnArgs &a, int g, const int64_t *map, int b, int quarter, bf16 *P1,
                           uint8_t *stage) {
    __shared__ int32_t s_slot[4];
    if (threadIdx.x < 4) s_slot[threadIdx.x] = a.records[map[b] * REC_INTS + g + threadIdx.x];
    __syncthreads();
    constexpr int F16 = FRAME_BYTES / 16;  // 441
    constexpr int PER = (4 * F16 + GEMM_THREADS - 1) / GEMM_THREADS;
    uint4 buf[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * GEMM_THREADS, c = e / F16, o = e - c * F16;
        buf[i] = make_uint4(0, 0, 0, 0);
        if (e < 4 * F16 && s_slot[c] >= 0)
            buf[i] = __ldg(reinterpret_cast<const uint4 *>(a.ring + (size_t)s_slot[c] * FRAME_BYTES) + o);
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * GEMM_THREADS;
        if (e < 4 * F16) reinterpret_cast<uint4 *>(stage)[e] = buf[i];
    }
    __syncthreads();
    bf16 *dst = P1 + (size_t)b * 400 * P1_LD;
    for (int e = quarter * 100 * 32 + threadIdx.x; e < (quarter + 1) * 100 * 32; e += GEMM_THREADS) {
        // 8-column chunk j of patch row `row` in the permuted K order (qnet.cuh w1_perm):
        // tap (ty, tx) = j >> 3, frame c = (j >> 1) & 3, rows dy0 = 2 (j & 1), dy0 + 1
        const int row = e >> 5, j = e & 31, tap = j >> 3, c = (j >> 1) & 3, dy0 = (j & 1) * 2;
        const int oy = row / 20, ox = row - oy * 20;
        const uint8_t *src = stage + c * FRAME_BYTES + (4 * oy + 4 * (tap >> 1) + dy0) * 84 + 4 * ox + 4 * (tap & 1);
        *reinterpret_cast<uint4 *>(dst + (size_t)row * P1_LD + j * 8) =
            u8x8_to_bf16(*reinterpret_cast<const uint32_t *>(src), *reinterpret_cast<const uint32_t *>(src + 84));
    }
    __syncthreads();
}

PQ_DEV void run_job(const Ctx &c, int type, int g, int uj, int j) {
    const PLearnArgs &a = *c.a;
    Pipe &P = *c.P;
    const int n = a.n, par = uj & 1;
    const int upd = c.u_base + uj;
    const int64_t *map = a.idx_base + (int64_t)upd * n;
    const pq_net &net = g ? a.target : a.theta;
    switch (type) {
        case J_G1:
            gather_patches(a, g, map, j >> 2, j & 3, a.P1[g][par], P.smem);
            break;
        case J_F1:  // conv1 8x8/4: P1 x W1^T, bias + ReLU with the 1/255 input scale
            tma_tile<32, false, false>(op(a, M_P1 + 2 * g + par, OP_K2, 2, j * 128), op(a, M_W1 + g, OP_K2, 1, 0),
                                       EpiConv1{a.wsb, g ? nullptr : a.act1, a.P2[g], net.master + P_B1, n, 1.0f / 255.0f},
                                       0, 4, j * 128, 0, 0, P);
            break;
        case J_F2:
            tma_tile<64, false, false>(op(a, M_P2 + g, OP_K2, 2, j * 128), op(a, M_W2 + g, OP_K2, 1, 0),
                                       EpiConv2{a.wsb, a.act2[g], net.master + P_B2, n}, 0, 8, j * 128, 0,
                                       0, P);
            break;
        case J_F3:
            tma_tile<64, false, false>(op(a, M_ACT2I + g, OP_IF3, 2, j * 128), op(a, M_W3 + g, OP_K2, 1, 0),
                                       EpiConv3{a.wsb, a.act3[g][par], net.master + P_B3, n}, 0, 9,
                                       j * 128, 0, 0, P);
            break;
        case J_F4: {  // fc1 swapped: D[j][b] = W4[j] . x[b], split-K partials [s][b][j]
            const Counts cn = counts_of(n);
            const int mt = j & 3, r = j >> 2, nt = r % cn.nt64, sp = r / cn.nt64;
            const int kb0 = sp * PL_FC1_KC, kb1 = min(49, kb0 + PL_FC1_KC);
            tma_tile<64, false, false>(op(a, M_W4 + g, OP_K2, 2, mt * 128),
                                       op(a, M_ACT3 + 2 * g + par, OP_K2, 1, nt * 64),
                                       EpiF32T{a.fc1part[g][par], 512, n, 512, (size_t)n * 512}, kb0, kb1, mt * 128,
                                       nt * 64, sp, P);
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
        case J_B4D: {  // D[b][k] = sum_j dh1[b][j] W4[j][k] (W4 as MN-major B)
            const int mt = j / 49, nt = j % 49;
            tma_tile<64, false, true>(op(a, M_DH1, OP_K2, 2, mt * 128), op(a, M_W4, OP_M2, 1, nt * 64),
                                      EpiB4D{a.wsb, a.dY3, a.act3[0][par], n}, 0, 8, mt * 128, nt * 64, 0, P);
            break;
        }
        case J_B3D:  // dY2 = relu'(x2) * transposed conv3(dY3): TP3 x W3 taps
            tma_tile<64, false, true>(op(a, M_DY3I, OP_IT3, 2, j * 128), op(a, M_W3V, OP_W3V, 1, 0),
                                      EpiB3D{a.wsb, a.dY2, a.act2[0], n}, 0, 9, j * 128, 0, 0, P);
            break;
        case J_B3W: {  // dW3^T[k][o] = sum_m P3[m][k] dY3[m][o]; column 576 = ones -> bias
            const int mt = j % 5, sp = j / 5;
            const int nch = (n * 49 + 63) / 64, kb0 = sp * a.kc3, kb1 = min(nch, kb0 + a.kc3);
            tma_tile<64, true, true>(op(a, M_ACT2W, OP_IW3, 2, mt * 128), op(a, M_DY3, OP_M2, 1, 0),
                                     EpiF32T{a.part3, 577, 64, 577, (size_t)64 * 577}, kb0, kb1, mt * 128, 0, sp, P);
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
            tma_tile<64, false, true>(op(a, M_DH1T, OP_K2, 2, mt * 128), op(a, M_ACT3 + par, OP_M2, 1, nt * 64), e,
                                      0, (n + 63) / 64, mt * 128, nt * 64, 0, P);
            break;
        }
        case J_B2D: {  // dY1 = relu'(x1) * transposed conv2(dY2), 4 input-parity classes
            const int tpc = counts_of(n).tpc, cls = j / tpc, loc = j - cls * tpc;
            tma_tile<64, false, true>(op(a, M_DY2I, OP_IT2, 2, loc * 128), op(a, M_W2V, OP_W2V, 1, 0, cls),
                                      EpiB2D{a.wsb, a.dY1, a.act1, n, tpc}, 0, 4, j * 128, 0, 0, P);
            break;
        }
        case J_B2W: {
            const int mt = j % 5, sp = j / 5;
            const int nch = (n * 81 + 63) / 64, kb0 = sp * a.kc2, kb1 = min(nch, kb0 + a.kc2);
            tma_tile<64, true, true>(op(a, M_P2, OP_M2, 2, mt * 128), op(a, M_DY2, OP_M2, 1, 0),
                                     EpiF32T{a.part2, 513, 64, 513, (size_t)64 * 513}, kb0, kb1, mt * 128, 0, sp, P);
            break;
        }
        case J_B1W: {  // dW1^T[k][o] = sum_m P1[m][k] dY1[m][o]; column 256 = ones
            const int mt = j % 3, sp = j / 3;
            const int nch = (n * 400 + 63) / 64, kb0 = sp * a.kc1, kb1 = min(nch, kb0 + a.kc1);
            tma_tile<64, true, true>(op(a, M_P1 + par, OP_M2, 2, mt * 128), op(a, M_DY1, OP_M2, 1, 0),
                                     EpiF32T{a.part1, 257, 32, 257, (size_t)32 * 257}, kb0, kb1, mt * 128, 0, sp, P);
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
            o.w1_perm = 1;  // conv1 weight-gradient rows in the permuted K order
            const int64_t lo = opt_lo(type) + (int64_t)j * PL_OPT_PER_JOB;
            const int64_t hi = min(opt_hi(type, a.A), lo + PL_OPT_PER_JOB);
            for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) opt_param(o, i, upd);
            break;
        }
    }
}

// the idx-th job of the critical (filler = 0) or filler (1) list of the phase
PQ_DEV void run_listed(const Ctx &c, const PhasePlan &P, int u, int filler, int idx) {
    const PLearnArgs &a = *c.a;
    for (int s = 0; s < P.nseg; ++s) {
        const Seg &g = P.seg[s];
        if (g.filler != filler || u + g.du < 0 || u + g.du >= a.n_updates) continue;
        const int cnt = g.end - g.begin;
        if (idx < cnt) {
            const unsigned long long t0 = a.trace ? gtime() : 0ull;
            run_job(c, g.type, g.grp, u + g.du, g.begin + idx);
            if (a.trace && threadIdx.x == 0) {  // last job of this CTA in the phase
                unsigned long long *t = a.trace + ((size_t)c.k * gridDim.x + blockIdx.x) * 4;
                t[2] = (unsigned long long)g.type;
                t[3] = gtime() - t0;
            }
            return;
        }
        idx -= cnt;
    }
}

// Critical jobs are dealt round-robin over all CTAs; fillers round-robin over the CTAs
// left without a critical job (over all CTAs when there are none).
PQ_DEV void run_phase(const Ctx &c, const PhasePlan &P, int u) {
    const PLearnArgs &a = *c.a;
    int ncrit = 0, nfill = 0;
    for (int s = 0; s < P.nseg; ++s) {
        const Seg &g = P.seg[s];
        if (u + g.du < 0 || u + g.du >= a.n_updates) continue;
        (g.filler ? nfill : ncrit) += g.end - g.begin;
    }
    const int G = gridDim.x, me = blockIdx.x;
    for (int j = me; j < ncrit; j += G) run_listed(c, P, u, 0, j);
    if (ncrit < G) {
        if (me >= ncrit)
            for (int f = me - ncrit; f < nfill; f += G - ncrit) run_listed(c, P, u, 1, f);
    } else {
        for (int f = ((me - ncrit) % G + G) % G; f < nfill; f += G) run_listed(c, P, u, 1, f);
    }
}

// one phase, then the grid barrier (with the optional trace rows)
PQ_DEV void run_phase_sync(Ctx &c, const PhasePlan &PP, int u, unsigned &target) {
    const PLearnArgs &a = *c.a;
    run_phase(c, PP, u);
    if (a.trace && threadIdx.x == 0) a.trace[((size_t)c.k * gridDim.x + blockIdx.x) * 4] = gtime();
    grid_barrier(a.bar, target);
    if (a.trace && threadIdx.x == 0) a.trace[((size_t)c.k * gridDim.x + blockIdx.x) * 4 + 1] = gtime();
    ++c.k;
}

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_learn_persistent(const __grid_constant__ PLearnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[PL_STAGES], empty[PL_STAGES], accb;
    __shared__ uint32_t tmem_base_s;
    __shared__ int s_ubase;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) {
        for (int s = 0; s < PL_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&accb, 1);
        fence_mbar_init();
        s_ubase = *a.update_counter;
    }
    if ((threadIdx.x >> 5) == 0) tmem_alloc<64>(&tmem_base_s);
    if (threadIdx.x < M_COUNT)
        asm volatile("prefetch.tensormap [%0];" ::"l"(&a.maps[threadIdx.x]) : "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    Pipe P{smem, smem_u32(smem), full, empty, &accb, 0u, 0u, &tmem_base_s};
    Ctx c{&a, &P, s_ubase, 0};
    unsigned target = 0;
    {
        const Sched &S = a.sched[SCHED_PROLOGUE];
        for (int p = 0; p < S.nphases; ++p) run_phase_sync(c, S.ph[p], 0, target);
    }
    for (int u = 0; u < a.n_updates; ++u) {
        const Sched &S = a.sched[u == a.n_updates - 1 ? SCHED_LAST : SCHED_STEADY];
        for (int p = 0; p < S.nphases; ++p) run_phase_sync(c, S.ph[p], u, target);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.update_counter = s_ubase + a.n_updates;
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) tmem_dealloc<64>(tmem_base_s);
}

// constant ones of the online operands of the weight-gradient GEMMs (bias gradients):
// P1 column 256, P2 column 512 and column 0 of the [64][64] ones tile; everything else
// never written stays zero from the allocation
__global__ void k_plearn_ones(bf16 *P1a, bf16 *P1b, bf16 *P2, bf16 *ones, int n) {
    const bf16 one = __float2bfloat16_rn(1.0f);
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n * 400; r += gridDim.x * blockDim.x) {
        P1a[(size_t)r * P1_LD + 256] = one;
        P1b[(size_t)r * P1_LD + 256] = one;
        if (r < n * 81) P2[(size_t)r * P2_LD + 512] = one;
        if (r < 64) ones[r * 64] = one;
    }
}

// ------------------------------------------------------------------ host side
static size_t al(size_t x) { return (x + 1023) & ~size_t(1023); }

struct PWS {
    bf16 *act1, *act2[2], *act3[2][2];
    bf16 *ones;  // [64][64], column 0 = 1: the bias-gradient atom of the conv3 wgrad
    bf16 *P1[2][2], *P2[2];
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
    w.act1 = (bf16 *)take((size_t)N * 400 * 32 * 2);
    for (int g = 0; g < 2; ++g) {
        w.act2[g] = (bf16 *)take((size_t)N * 81 * 64 * 2);
        for (int p = 0; p < 2; ++p) {
            w.act3[g][p] = (bf16 *)take((size_t)N * 3136 * 2);
            w.P1[g][p] = (bf16 *)take((size_t)N * 400 * P1_LD * 2);
            w.fc1part[g][p] = (float *)take((size_t)PL_FC1_SPLITS * N * 512 * 4);
        }
        w.P2[g] = (bf16 *)take((size_t)N * 81 * P2_LD * 2);
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
    w.ones = (bf16 *)take(64 * 64 * 2);
    w.part1 = (float *)take((size_t)MAX_SPLITS * 32 * 257 * 4);
    w.part2 = (float *)take((size_t)MAX_SPLITS * 64 * 513 * 4);
    w.part3 = (float *)take((size_t)MAX_SPLITS * 64 * 577 * 4);
    w.bar = (unsigned *)take(sizeof(unsigned));
    w.bytes = off;
    return w;
}

// ---- tensor maps (driver entry point; no -lcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
    static void *fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

// bf16 tensor of `rank` dims (innermost first), strides of dims 1.. in elements;
// boxes of 64 elements (128 B, 128B swizzle) x 1 x .. x `outer_box` rows of the outermost
// dim (64 for tiles, 1 for gather4 row maps)
static int make_map(CUtensorMap *m, const void *base, int rank, const uint64_t *dims, const uint64_t *strides_el,
                    const char *what, uint32_t outer_box = 64) {
    auto enc = encode_tiled();
    if (!enc) return set_err("cuTensorMapEncodeTiled unavailable (driver entry point)");
    cuuint64_t gd[5], gs[4];
    cuuint32_t box[5], es[5];
    for (int i = 0; i < rank; ++i) {
        gd[i] = dims[i];
        es[i] = 1;
        box[i] = i == 0 ? 64 : i == rank - 1 ? outer_box : 1;
        if (i > 0) gs[i - 1] = strides_el[i - 1] * 2;
    }
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(base), gd, gs, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char msg[160];
        snprintf(msg, sizeof(msg), "tensor map %s: CUresult %d", what, (int)r);
        return set_err(msg);
    }
    return 0;
}
static int map2(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols, uint64_t ld, const char *what) {
    const uint64_t dims[2] = {cols, rows}, st[1] = {ld};
    return make_map(m, base, 2, dims, st, what);
}
static PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col() {
    static void *fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
}

// im2col map of an NHWC bf16 tensor [n][H][W][64]: `pixels` pixels x 64 channels per
// load; base pixels range over [lo, W-1+hi] x [lo, H-1+hi] (corners in W, H order)
static int map_im2col(CUtensorMap *m, const void *base, int n, int H, int W, int lo, int hi, int pixels,
                      const char *what, int C = 64) {
    auto enc = encode_im2col();
    if (!enc) return set_err("cuTensorMapEncodeIm2col unavailable (driver entry point)");
    const cuuint64_t gd[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
    const cuuint64_t gs[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    const int lower[2] = {lo, lo}, upper[2] = {hi, hi};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), gd, gs, lower, upper, 64,
                     (cuuint32_t)pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char msg[160];
        snprintf(msg, sizeof(msg), "im2col tensor map %s: CUresult %d", what, (int)r);
        return set_err(msg);
    }
    return 0;
}

static int build_maps(PLearnArgs &a) {
    const int n = a.n;
    for (int g = 0; g < 2; ++g) {
        const bf16 *sh = (const bf16 *)(g ? a.target.shadow : a.theta.shadow);
        if (int rc = map2(&a.maps[M_W1 + g], sh + S_W1P, 32, 256, 256, "W1 permuted")) return rc;
        if (int rc = map2(&a.maps[M_W2 + g], sh + S_W2, 64, 512, 512, "W2")) return rc;
        if (int rc = map2(&a.maps[M_W3 + g], sh + S_W3, 64, 576, 576, "W3")) return rc;
        if (int rc = map2(&a.maps[M_W4 + g], sh + S_W4, 512, 3136, 3136, "W4")) return rc;
        for (int p = 0; p < 2; ++p) {
            if (int rc = map2(&a.maps[M_ACT3 + 2 * g + p], a.act3[g][p], n, 3136, 3136, "act3")) return rc;
            if (int rc = map2(&a.maps[M_P1 + 2 * g + p], a.P1[g][p], (uint64_t)n * 400, 257, P1_LD, "P1")) return rc;
        }
        if (int rc = map2(&a.maps[M_P2 + g], a.P2[g], (uint64_t)n * 81, 513, P2_LD, "P2")) return rc;
        if (int rc = map_im2col(&a.maps[M_ACT2I + g], a.act2[g], n, 9, 9, 0, -2, 128, "act2")) return rc;
    }
    if (int rc = map_im2col(&a.maps[M_ACT2W], a.act2[0], n, 9, 9, 0, -2, 64, "act2 wgrad")) return rc;
    if (int rc = map_im2col(&a.maps[M_DY3I], a.dY3, n, 7, 7, -2, 0, 128, "dY3")) return rc;
    if (int rc = map_im2col(&a.maps[M_DY2I], a.dY2, n, 9, 9, -1, 0, 128, "dY2")) return rc;
    if (int rc = map2(&a.maps[M_ONES], a.ones, 64, 64, 64, "ones")) return rc;
    if (int rc = map2(&a.maps[M_DH1], a.dh1_bf, n, 512, 512, "dh1")) return rc;
    if (int rc = map2(&a.maps[M_DH1T], a.dh1T, 512, n, a.n8, "dh1T")) return rc;
    if (int rc = map2(&a.maps[M_DY3], a.dY3, (uint64_t)n * 49, 64, 64, "dY3")) return rc;
    if (int rc = map2(&a.maps[M_DY2], a.dY2, (uint64_t)n * 81, 64, 64, "dY2")) return rc;
    if (int rc = map2(&a.maps[M_DY1], a.dY1, (uint64_t)n * 400, 32, 32, "dY1")) return rc;
    const bf16 *sh = (const bf16 *)a.theta.shadow;
    {  // conv3 weight [o][kh][kw][c] as (c, tap, o)
        const uint64_t dims[3] = {64, 9, 64}, st[2] = {64, 576};
        if (int rc = make_map(&a.maps[M_W3V], sh + S_W3, 3, dims, st, "W3 view")) return rc;
    }
    {  // conv2 weight [o][kh][kw][c] as (c, kw, kh, o)
        const uint64_t dims[4] = {32, 4, 4, 64}, st[3] = {32, 128, 512};
        if (int rc = make_map(&a.maps[M_W2V], sh + S_W2, 4, dims, st, "W2 view")) return rc;
    }
    return 0;
}

// split-K factor for `mtiles` M tiles of a contraction of `nch` 64-wide chunks given a
// CTA budget: chunks per split >= 2, splits <= MAX_SPLITS
static void choose_split(int nch, int mtiles, int budget, int *kc, int *splits) {
    int s = std::max(1, budget / mtiles);
    int k = std::max(2, (nch + s - 1) / s);
    k = std::max(k, (nch + MAX_SPLITS - 1) / MAX_SPLITS);
    *kc = k;
    *splits = (nch + k - 1) / k;
}

struct PlanBuilder {
    Sched &S;
    int n, A, s1, s2, s3;
    int count(int type) const { return njobs(type, n, A, s1, s2, s3); }
    void add(int p, int type, int grp, int du, int filler, int begin = 0, int end = -1) {
        if (end < 0) end = count(type);
        if (end <= begin) return;
        PhasePlan &P = S.ph[p];
        P.seg[P.nseg++] = Seg{(int16_t)type, (int8_t)grp, (int8_t)du, (int16_t)filler, 0, begin, end};
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
    choose_split((n * 400 + 63) / 64, 3, G, &a.kc1, &a.s1);
    choose_split((n * 81 + 63) / 64, 5, std::max(5, G - 4 * cn.tpc), &a.kc2, &a.s2);
    choose_split((n * 49 + 63) / 64, 5, std::max(5, G - cn.t2), &a.kc3, &a.s3);
    {  // prologue: frame gathers of steps 0 / 1 and the target forward of step 0
        PlanBuilder b{a.sched[SCHED_PROLOGUE], n, A, a.s1, a.s2, a.s3};
        b.add(0, J_G1, 1, 0, 0);
        b.add(0, J_G1, 0, 0, 0);
        b.add(0, J_G1, 1, +1, 0);
        b.add(1, J_F1, 1, 0, 0);
        b.add(2, J_F2, 1, 0, 0);
        b.add(3, J_F3, 1, 0, 0);
        b.add(4, J_F4, 1, 0, 0);
    }
    for (int last = 0; last < 2; ++last) {
        PlanBuilder b{a.sched[last ? SCHED_LAST : SCHED_STEADY], n, A, a.s1, a.s2, a.s3};
        // the critical chain of the step
        b.add(0, J_F1, 0, 0, 0);
        b.add(1, J_F2, 0, 0, 0);
        b.add(2, J_F3, 0, 0, 0);
        b.add(3, J_F4, 0, 0, 0);
        b.add(4, J_HEAD, 0, 0, 0);
        b.add(5, J_B4D, 0, 0, 0);
        b.add(6, J_B3D, 0, 0, 0);
        b.add(6, J_B3W, 0, 0, 0);
        b.add(7, J_B2D, 0, 0, 0);
        b.add(7, J_B2W, 0, 0, 0);
        b.add(8, J_B1W, 0, 0, 0);
        b.add(9, J_OPT_C1, 0, 0, 0);
        b.add(9, J_OPT_C2, 0, 0, 0);
        b.add(9, J_OPT_C3, 0, 0, 0);
        // fillers: next steps' target forward and frame gathers (skipped past the
        // launch's end), the fc2 / fc1-bias update
        b.add(1, J_F1, 1, +1, 1);
        b.add(2, J_F2, 1, +1, 1);
        b.add(3, J_F3, 1, +1, 1);
        b.add(4, J_F4, 1, +1, 1);
        b.add(5, J_OPT_FC2, 0, 0, 1);
        b.add(5, J_G1, 1, +2, 1);
        b.add(9, J_G1, 0, +1, 1);
    }
    // fc1 weight gradient + RMSProp tiles into the spare CTAs of the phases where they
    // may run: 6-9 of their own step, 0-2 of the next (du = -1 there).  The split is
    // decided for a steady step; the last step of a launch runs the previous step's
    // leftovers in 0-2 as usual and all of its own tiles in 6-9.
    PlanBuilder st{a.sched[SCHED_STEADY], n, A, a.s1, a.s2, a.s3};
    PlanBuilder ls{a.sched[SCHED_LAST], n, A, a.s1, a.s2, a.s3};
    const int total = st.count(J_B4W);
    const int own[3] = {6, 7, 8}, nxt[3] = {0, 1, 2};
    int next = 0;
    for (int p : own) {
        const int take = std::min(total - next, std::max(0, G - st.load(p)));
        if (take > 0) st.add(p, J_B4W, 0, 0, 1, next, next + take);
        next += std::max(0, take);
    }
    for (int p : nxt) {
        const int take = std::min(total - next, std::max(0, G - st.load(p)));
        if (take > 0) {
            st.add(p, J_B4W, 0, -1, 1, next, next + take);
            ls.add(p, J_B4W, 0, -1, 1, next, next + take);
        }
        next += std::max(0, take);
    }
    if (next < total) st.add(9, J_B4W, 0, 0, 1, next, total);
    next = 0;
    for (int p : own) {
        const int take = std::min(total - next, std::max(0, G - ls.load(p)));
        if (take > 0) ls.add(p, J_B4W, 0, 0, 1, next, next + take);
        next += std::max(0, take);
    }
    if (next < total) ls.add(9, J_B4W, 0, 0, 1, next, total);
}

// ================================================================== one-shot TMA GEMMs
// The learner-step GEMMs of the CUDA-graph path (qnet.cu) on the TMA engine: one CTA per
// SM loops over the output tiles of ONE GEMM (up to 2 parameter groups), keeping its
// TMEM, ring and barriers across tiles; operands as TmaOp (tiled boxes / im2col).
template <class EP>
struct TmaGemm {
    CUtensorMap a[2], b[2], aux;
    EP ep[2];
    int kindA, kindB, boxesA, boxesB;
    int n, tpc;
    int mtiles, ntiles, splits, groups;
    int kc, nk;       // K-chunks per split, total K-chunks
    int b_is_weight;  // B never comes from the preceding kernel: prefetched before the PDL wait
    int cls0[2];      // IF1: channel start of each group (16 g: frames g..g+3)
};

// Warp-specialised persistent tile loop (one CTA per SM):
//   warp 0      producer: streams every tile's operand boxes into the 6-slot ring,
//               running ahead across tile boundaries (slot reuse gated by `empty`);
//   warp 1      MMA issuer: alternates two 64-column TMEM accumulators; tile i waits
//               until the epilogue released the buffer of tile i-2 (`acce`), commits
//               each slot back to the producer and the finished accumulator (`accf`);
//   warps 4-7   epilogue: TMEM lane quadrant w-4 = tile rows 32(w-4).., read the
//               accumulator into registers, release it, then apply the fused epilogue
//               (staged epilogues use a dedicated 33 KB shared tile, not the ring),
// so tile t's epilogue overlaps tile t+1's loads and MMAs.
constexpr int TG_STAGES = 6;
constexpr int TG_STAGE_TILE = 128 * 65 * 4;  // fp32 staging tile of EpiRms (BN = 64)
constexpr int TG_SMEM = TG_STAGES * PL_SLOT + TG_STAGE_TILE + 1024;

template <class EP>
PQ_DEV void tg_decode(const TmaGemm<EP> &g, int t, int BN, TmaOp &A, TmaOp &B, int &kb0, int &kb1, int &m0,
                      int &n0, int &sp, int &grp) {
    const int per_grp = g.mtiles * g.ntiles * g.splits;
    grp = t / per_grp;
    const int r = t - grp * per_grp;
    const int mt = r % g.mtiles, r2 = r / g.mtiles, nt = r2 % g.ntiles;
    sp = r2 / g.ntiles;
    int r0 = mt * 128, cls = 0;
    if (g.kindA == OP_IT2) {  // class-major tiles: tpc tiles per input-parity class
        cls = mt / g.tpc;
        r0 = (mt - cls * g.tpc) * 128;
    }
    A = TmaOp{&g.a[grp], g.kindA, g.boxesA, r0, g.kindA == OP_IF1 ? g.cls0[grp] : cls, g.n, &g.aux};
    B = TmaOp{&g.b[grp], g.kindB, g.boxesB, nt * BN, cls, g.n, &g.aux};
    kb0 = sp * g.kc;
    kb1 = min(g.nk, kb0 + g.kc);
    m0 = mt * 128;
    n0 = nt * BN;
}

template <int BN, bool AMN, bool BMN, class EP>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_tma_gemm(const __grid_constant__ TmaGemm<EP> g) {
    TlProbe tp;
    static_assert(BN == 64, "the one-shot TMA GEMMs use 64-column accumulators");
    constexpr uint32_t IDESC = idesc_bf16(BN, AMN, BMN);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[TG_STAGES], empty[TG_STAGES], accf[2], acce[2];
    __shared__ uint32_t tmem_base_s;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t smem_s = smem_u32(smem);
    float *stage_tile = reinterpret_cast<float *>(smem + TG_STAGES * PL_SLOT);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < TG_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 4);  // one arrival per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<128>(&tmem_base_s);
    if (tid < 2 * g.groups) {
        const CUtensorMap *m = (tid & 1) ? &g.b[tid >> 1] : &g.a[tid >> 1];
        asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int total = g.mtiles * g.ntiles * g.splits * g.groups;
    // weights (never written by the preceding kernel) of the first tile's first chunks
    // are requested before the dependency wait, so they land while the predecessor drains
    int pre = 0;
    if (tid == 0 && g.b_is_weight && (int)blockIdx.x < total) {
        TmaOp A, B;
        int kb0, kb1, m0, n0, sp, grp;
        tg_decode(g, blockIdx.x, BN, A, B, kb0, kb1, m0, n0, sp, grp);
        const uint32_t bytes = (uint32_t)(A.boxes + B.boxes) * PL_BOX;
        for (int kb = kb0; kb < kb1 && pre < TG_STAGES; ++kb, ++pre) {
            mbar_expect_tx(&full[pre], bytes);
            B.issue(smem_s + pre * PL_SLOT + PL_B_OFF, &full[pre], kb, 0);
        }
    }
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                TmaOp A, B;
                int kb0, kb1, m0, n0, sp, grp;
                tg_decode(g, t, BN, A, B, kb0, kb1, m0, n0, sp, grp);
                const uint32_t bytes = (uint32_t)(A.boxes + B.boxes) * PL_BOX;
                for (int kb = kb0; kb < kb1; ++kb, ++q) {
                    const uint32_t s = q % TG_STAGES;
                    const uint32_t dst = smem_s + s * PL_SLOT;
                    if ((int)q < pre) {  // B already requested (and the slot armed) before the wait
                        A.issue(dst, &full[s], kb, 0);
                        continue;
                    }
                    if (q >= TG_STAGES) mbar_wait(&empty[s], ((q / TG_STAGES) - 1) & 1);
                    mbar_expect_tx(&full[s], bytes);
                    A.issue(dst, &full[s], kb, 0);
                    B.issue(dst + PL_B_OFF, &full[s], kb, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            uint32_t q = 0, it = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
                TmaOp A, B;
                int kb0, kb1, m0, n0, sp, grp;
                tg_decode(g, t, BN, A, B, kb0, kb1, m0, n0, sp, grp);
                const uint32_t buf = it & 1;
                if (it >= 2) mbar_wait(&acce[buf], ((it >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t acc = tmem + buf * BN;
                for (int kb = kb0; kb < kb1; ++kb, ++q) {
                    const uint32_t s = q % TG_STAGES;
                    mbar_wait(&full[s], (q / TG_STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a_addr = smem_s + s * PL_SLOT, b_addr = a_addr + PL_B_OFF;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t ad =
                            AMN ? desc_sw128(a_addr + j * 2048, 8192) : desc_sw128(a_addr + j * 32, 0);
                        const uint64_t bd =
                            BMN ? desc_sw128(b_addr + j * 2048, 8192) : desc_sw128(b_addr + j * 32, 0);
                        umma_bf16(acc, ad, bd, IDESC, (kb > kb0 || j > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&accf[buf]);
            }
        }
    } else if (warp >= 4) {  // epilogue
        const int wq = warp - 4;
        uint32_t it = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
            TmaOp A, B;
            int kb0, kb1, m0, n0, sp, grp;
            tg_decode(g, t, BN, A, B, kb0, kb1, m0, n0, sp, grp);
            const uint32_t buf = it & 1;
            mbar_wait(&accf[buf], (it >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            float v[2][32];
            const uint32_t trow = tmem + buf * BN + ((uint32_t)(wq * 32) << 16);
            if (kb1 > kb0) {
                tmem_ld32(trow, v[0]);
                tmem_ld32(trow + 32, v[1]);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[0][e] = v[1][e] = 0.f;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[buf]);
            const EP &ep = g.ep[grp];
            const int row = m0 + wq * 32 + lane;
            if constexpr (is_staged<EP>::value) {
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) stage_tile[(wq * 32 + lane) * (BN + 1) + c * 32 + e] = v[c][e];
                named_bar_sync(1, 128);
                ep.template apply_tile_w<BN, 4>(stage_tile, BN + 1, m0, n0, wq);
                named_bar_sync(1, 128);
            } else {
                ep.apply(row, n0, v[0], 32, sp);
                ep.apply(row, n0 + 32, v[1], 32, sp);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
    tp.done('T');
}

static int g_sms = 0;
template <int BN, bool AMN, bool BMN, class EP>
static int launch_tma(const TmaGemm<EP> &g, cudaStream_t st, const char *what) {
    auto kern = k_tma_gemm<BN, AMN, BMN, EP>;
    static bool configured = false;  // per instantiation
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TG_SMEM));
        configured = true;
    }
    if (!g_sms) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int total = g.mtiles * g.ntiles * g.splits * g.groups;
    return cuda_err(launch_k(kern, dim3(std::min(total, g_sms)), dim3(GEMM_THREADS), TG_SMEM, st, g), what);
}

// the [64][64] ones tile (column 0 = 1): bias-gradient atom of the conv3 wgrad
__global__ void k_ones_tile(bf16 *t) {
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) t[i] = __float2bfloat16_rn((i & 63) == 0 ? 1.f : 0.f);
}
static bf16 *ones_tile(cudaStream_t st) {
    static bf16 *t = nullptr;
    if (!t) {
        if (cudaMalloc(&t, 64 * 64 * 2) != cudaSuccess) return nullptr;
        k_ones_tile<<<1, 256, 0, st>>>(t);
    }
    return t;
}

// conv3 forward, groups online / target: act3[g] = relu(im2col(act2[g]) W3[g]^T + b3[g])
int tma_conv3_fwd(const pq_net *nets, bf16 *const *act2, bf16 *const *act3, int groups, int n, cudaStream_t st) {
    static thread_local TmaGemm<EpiBiasRelu> g;  // per host thread (launch arguments are copied at launch)
    memset(&g, 0, sizeof(g));
    for (int q = 0; q < groups; ++q) {
        if (int rc = map_im2col(&g.a[q], act2[q], n, 9, 9, 0, -2, 128, "act2")) return rc;
        if (int rc = map2(&g.b[q], (const bf16 *)nets[q].shadow + S_W3, 64, 576, 576, "W3")) return rc;
        g.ep[q] = EpiBiasRelu{act3[q], nets[q].master + P_B3, n * 49, 64, 64, 1.0f};
    }
    g.kindA = OP_IF3, g.kindB = OP_K2, g.boxesA = 2, g.boxesB = 1, g.n = n, g.b_is_weight = 1;
    g.mtiles = (n * 49 + 127) / 128, g.ntiles = 1, g.splits = 1, g.groups = groups, g.kc = 9, g.nk = 9;
    return launch_tma<64, false, false>(g, st, "conv3 forward (TMA)");
}

// fc1 forward, swapped: part[g][s][b][j] = sum over split s of W4[g][j] . act3[g][b]
int tma_fc1_fwd(const pq_net *nets, bf16 *const *act3, float *const *part, int splits, int groups, int n,
                cudaStream_t st) {
    static thread_local TmaGemm<EpiF32T> g;
    memset(&g, 0, sizeof(g));
    for (int q = 0; q < groups; ++q) {
        if (int rc = map2(&g.a[q], (const bf16 *)nets[q].shadow + S_W4, 512, 3136, 3136, "W4")) return rc;
        if (int rc = map2(&g.b[q], act3[q], n, 3136, 3136, "act3")) return rc;
        g.ep[q] = EpiF32T{part[q], 512, n, 512, (size_t)n * 512};
    }
    g.kindA = OP_K2, g.kindB = OP_K2, g.boxesA = 2, g.boxesB = 1, g.n = n;
    g.mtiles = 4, g.ntiles = (n + 63) / 64, g.splits = splits, g.groups = groups;
    g.nk = 49, g.kc = (49 + splits - 1) / splits;
    return launch_tma<64, false, false>(g, st, "fc1 forward (TMA)");
}

// ---- fc1 GEMMs with the A operand resident (large batches)
// One CTA per (group, 128-row M tile, K split, N range) keeps all its A chunks in shared
// memory and streams only the B tiles of its N range, so A is read once per CTA instead of
// once per 64-wide N tile.  Per output tile the same K chunks in the same order as the
// k_tma_gemm version, so results are bit-identical.
//  * fc1 forward (swapped): A = W4 [512][3136] (7 chunks per split, 112 KB, requested
//    before the dependency wait), B = act3 (K-major), EpiF32T split partials;
//  * fc1 data gradient: A = dh1 [n][512] (8 chunks, 128 KB; written by the head, so after
//    the wait), B = W4 as MN-major [512][3136], EpiMask (relu' of act3).
constexpr int RA_MAXKC = 8, RA_STAGES = 4;
constexpr int RA_SMEM = 1024 + RA_MAXKC * 2 * PL_BOX + RA_STAGES * PL_BOX;
template <class EP>
struct RAArgs {
    CUtensorMap a[2], b[2];
    EP ep[2];
    int groups, mtiles, ntiles, splits, nparts, nk, kc, a_early;
};

template <class EP, bool BMN>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_resident_a(const __grid_constant__ RAArgs<EP> g) {
    constexpr uint32_t IDESC = idesc_bf16(64, false, BMN);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[RA_STAGES], empty[RA_STAGES], accf[2], acce[2], abar;
    __shared__ uint32_t tmem_base_s;
    TlProbe tp;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t a_s = smem_u32(smem), ring_s = a_s + RA_MAXKC * 2 * PL_BOX;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int t = blockIdx.x;  // -> (group, M tile, split, N range)
    const int part = t % g.nparts;
    t /= g.nparts;
    const int split = t % g.splits;
    t /= g.splits;
    const int mt = t % g.mtiles, grp = t / g.mtiles;
    const int per = (g.ntiles + g.nparts - 1) / g.nparts;
    const int nt0 = part * per, nt1 = min(g.ntiles, nt0 + per);
    const int kb0 = split * g.kc, kb1 = min(g.nk, kb0 + g.kc), nk = kb1 - kb0;
    if (tid == 0) {
        for (int s = 0; s < RA_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 4);
        }
        mbar_init(&abar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<128>(&tmem_base_s);
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a[grp]) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.b[grp]) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    auto load_a = [&] {
        mbar_expect_tx(&abar, (uint32_t)(nk * 2 * PL_BOX));
        for (int c = 0; c < nk; ++c)
            for (int h = 0; h < 2; ++h)
                tma_load_2d(a_s + (c * 2 + h) * PL_BOX, &g.a[grp], &abar, (kb0 + c) * 64, mt * 128 + h * 64);
    };
    if (tid == 0 && nk > 0 && g.a_early) load_a();
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0 && nk > 0) {  // producer: A once (unless early), then B tile (n-tile, chunk) per slot
            if (!g.a_early) load_a();
            uint32_t q = 0;
            for (int nt = nt0; nt < nt1; ++nt)
                for (int c = 0; c < nk; ++c, ++q) {
                    const uint32_t s = q % RA_STAGES;
                    if (q >= RA_STAGES) mbar_wait(&empty[s], ((q / RA_STAGES) - 1) & 1);
                    mbar_expect_tx(&full[s], (uint32_t)PL_BOX);
                    if (BMN)
                        tma_load_2d(ring_s + s * PL_BOX, &g.b[grp], &full[s], nt * 64, (kb0 + c) * 64);
                    else
                        tma_load_2d(ring_s + s * PL_BOX, &g.b[grp], &full[s], (kb0 + c) * 64, nt * 64);
                }
        }
    } else if (warp == 1) {
        if (lane == 0 && nk > 0) {  // MMA issuer
            mbar_wait(&abar, 0);
            uint32_t q = 0, it = 0;
            for (int nt = nt0; nt < nt1; ++nt, ++it) {
                const uint32_t buf = it & 1, acc = tmem + buf * 64;
                if (it >= 2) mbar_wait(&acce[buf], ((it >> 1) - 1) & 1);
                tc_fence_after();
                for (int c = 0; c < nk; ++c, ++q) {
                    const uint32_t s = q % RA_STAGES;
                    mbar_wait(&full[s], (q / RA_STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a_addr = a_s + c * 2 * PL_BOX, b_addr = ring_s + s * PL_BOX;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t bd = BMN ? desc_sw128(b_addr + j * 2048, 8192) : desc_sw128(b_addr + j * 32, 0);
                        umma_bf16(acc, desc_sw128(a_addr + j * 32, 0), bd, IDESC, (c > 0 || j > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&accf[buf]);
            }
        }
    } else if (warp >= 4 && nk > 0) {  // epilogue
        const int wq = warp - 4;
        uint32_t it = 0;
        for (int nt = nt0; nt < nt1; ++nt, ++it) {
            const uint32_t buf = it & 1;
            mbar_wait(&accf[buf], (it >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            float v[2][32];
            const uint32_t trow = tmem + buf * 64 + ((uint32_t)(wq * 32) << 16);
            tmem_ld32(trow, v[0]);
            tmem_ld32(trow + 32, v[1]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[buf]);
            const int row = mt * 128 + wq * 32 + lane;
            g.ep[grp].apply(row, nt * 64, v[0], 32, split);
            g.ep[grp].apply(row, nt * 64 + 32, v[1], 32, split);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
    tp.done('4');
}

template <class EP, bool BMN>
static int launch_resident_a(RAArgs<EP> &g, cudaStream_t st, const char *what) {
    auto kern = k_resident_a<EP, BMN>;
    static bool configured = false;  // per instantiation
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RA_SMEM));
        configured = true;
    }
    if (!g_sms) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (g.kc > RA_MAXKC) return set_err("resident-A GEMM: too many K chunks per split");
    const int base = g.groups * g.mtiles * g.splits;
    g.nparts = std::max(1, std::min(g.ntiles, g_sms / base));  // one wave of CTAs
    return cuda_err(launch_k(kern, dim3(base * g.nparts), dim3(GEMM_THREADS), RA_SMEM, st, g), what);
}

int tma_fc1_fwd_resident(const pq_net *nets, bf16 *const *act3, float *const *part, int splits, int groups, int n,
                         cudaStream_t st) {
    static thread_local RAArgs<EpiF32T> g;
    memset(&g, 0, sizeof(g));
    for (int q = 0; q < groups; ++q) {
        if (int rc = map2(&g.a[q], (const bf16 *)nets[q].shadow + S_W4, 512, 3136, 3136, "W4")) return rc;
        if (int rc = map2(&g.b[q], act3[q], n, 3136, 3136, "act3")) return rc;
        g.ep[q] = EpiF32T{part[q], 512, n, 512, (size_t)n * 512};
    }
    g.groups = groups, g.mtiles = 4, g.ntiles = (n + 63) / 64, g.splits = splits, g.nk = 49;
    g.kc = (49 + splits - 1) / splits, g.a_early = 1;  // W4: updated two or more launches back
    return launch_resident_a<EpiF32T, false>(g, st, "fc1 forward (resident W4)");
}

int tma_fc1_dgrad_resident(const pq_net &th, const bf16 *dh1_bf, const bf16 *act3, bf16 *dY3, int n,
                           cudaStream_t st, bf16 *dY3p) {
    auto setup = [&](auto &g) -> int {
        memset(&g, 0, sizeof(g));
        if (int rc = map2(&g.a[0], dh1_bf, n, 512, 512, "dh1")) return rc;
        if (int rc = map2(&g.b[0], (const bf16 *)th.shadow + S_W4, 512, 3136, 3136, "W4")) return rc;
        g.groups = 1, g.mtiles = (n + 127) / 128, g.ntiles = 49, g.splits = 1, g.nk = 8, g.kc = 8, g.a_early = 0;
        return 0;
    };
    if (dY3p) {  // also onto the padded 11 x 11 grid of the shifted conv3 data gradient
        static thread_local RAArgs<EpiMaskPad7> g;
        if (int rc = setup(g)) return rc;
        g.ep[0] = EpiMaskPad7{EpiMask{dY3, act3, n, 3136, 3136}, dY3p};
        return launch_resident_a<EpiMaskPad7, true>(g, st, "fc1 dgrad (resident dh1, padded copy)");
    }
    static thread_local RAArgs<EpiMask> g;
    if (int rc = setup(g)) return rc;
    g.ep[0] = EpiMask{dY3, act3, n, 3136, 3136};
    return launch_resident_a<EpiMask, true>(g, st, "fc1 dgrad (resident dh1)");
}

// ---- conv3 data gradient by row-shifted descriptors
// dY2 = relu'(act2) * transposed conv3(dY3): on the zero-padded 11 x 11 grid dY3p (dY3 at
// (y + 2, x + 2), written by fc1's data gradient) GEMM row r = (s, y, x) (y, x = 9, 10
// discarded) reads row r + 11 (2 - kh) + (2 - kw) for tap (kh, kw); one TMA box of 152 rows
// feeds the 9 taps against 9 resident MN-major W3 tiles, in the tap order of the im2col
// kernel, so dY2 (and its padded copies) are bit-identical.
constexpr int C3D_ROWS = 152, C3D_BOX = C3D_ROWS * 128, C3D_STAGES = 3, C3D_W = 64 * 128;
constexpr int C3D_SMEM = 1024 + 9 * C3D_W + C3D_STAGES * C3D_BOX;
struct C3DArgs {
    CUtensorMap a, w;  // dY3p pixel rows [n*121][64]; W3 view {c, tap, o}
    EpiMaskPad ep;     // dY2 [n*81][64] + padded copies
    int n;
};

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_conv3_dgrad_shift(const __grid_constant__ C3DArgs g) {
    constexpr uint32_t IDESC = idesc_bf16(64, false, true);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[C3D_STAGES], empty[C3D_STAGES], accf[2], acce[2], wbar;
    __shared__ uint32_t tmem_base_s;
    TlProbe tp;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(smem), ring_s = w_s + 9 * C3D_W;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < C3D_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 4);
        }
        mbar_init(&wbar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<128>(&tmem_base_s);
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.w) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int total = (g.n * 121 + 127) / 128;
    if (tid == 0) {  // W3 (updated two or more launches back) before the dependency wait
        mbar_expect_tx(&wbar, 9u * C3D_W);
        for (int tap = 0; tap < 9; ++tap) tma_load_3d(w_s + tap * C3D_W, &g.w, &wbar, 0, tap, 0);
    }
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t s = q % C3D_STAGES;
                if (q >= C3D_STAGES) mbar_wait(&empty[s], ((q / C3D_STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], (uint32_t)C3D_BOX);
                tma_load_2d(ring_s + s * C3D_BOX, &g.a, &full[s], 0, t * 128);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            mbar_wait(&wbar, 0);
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t buf = q & 1, s = q % C3D_STAGES;
                if (q >= 2) mbar_wait(&acce[buf], ((q >> 1) - 1) & 1);
                mbar_wait(&full[s], (q / C3D_STAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = ring_s + s * C3D_BOX, acc = tmem + buf * 64;
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint32_t shift = (uint32_t)((2 - tap / 3) * 11 + (2 - tap % 3)) * 128;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t ad = desc_sw128(a0 + shift + j * 32, 0);
                        const uint64_t bd = desc_sw128(w_s + tap * C3D_W + j * 2048, 8192);
                        umma_bf16(acc, ad, bd, IDESC, (tap > 0 || j > 0) ? 1u : 0u);
                    }
                }
                umma_commit(&empty[s]);
                umma_commit(&accf[buf]);
            }
        }
    } else if (warp >= 4) {  // epilogue
        const int wq = warp - 4;
        uint32_t q = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
            const uint32_t buf = q & 1;
            mbar_wait(&accf[buf], (q >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            float v[2][32];
            const uint32_t trow = tmem + buf * 64 + ((uint32_t)(wq * 32) << 16);
            tmem_ld32(trow, v[0]);
            tmem_ld32(trow + 32, v[1]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[buf]);
            const int r = t * 128 + wq * 32 + lane, smp = r / 121, p = r - smp * 121, y = p / 11, x = p - y * 11;
            if (smp < g.n && y < 9 && x < 9) {
                const int m = smp * 81 + y * 9 + x;
                g.ep.apply(m, 0, v[0], 32, 0);
                g.ep.apply(m, 32, v[1], 32, 0);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
    tp.done('C');
}

int tma_conv3_dgrad_shift(const pq_net &th, const bf16 *dY3p, const bf16 *act2, bf16 *dY2, bf16 *dY2p, bf16 *dY2q,
                          int n, cudaStream_t st) {
    static thread_local C3DArgs g;
    memset(&g, 0, sizeof(g));
    const uint64_t ad[2] = {64, (uint64_t)n * 121}, as[1] = {64};
    if (int rc = make_map(&g.a, dY3p, 2, ad, as, "dY3 padded rows", C3D_ROWS)) return rc;
    const uint64_t dims[3] = {64, 9, 64}, strd[2] = {64, 576};
    if (int rc = make_map(&g.w, (const bf16 *)th.shadow + S_W3, 3, dims, strd, "W3 view")) return rc;
    g.ep = EpiMaskPad{EpiMask{dY2, act2, n * 81, 64, 64}, dY2p, FastDiv(81), FastDiv(9), dY2q};
    g.n = n;
    static bool configured = false;
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_conv3_dgrad_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, C3D_SMEM));
        configured = true;
    }
    if (!g_sms) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int total = (n * 121 + 127) / 128;
    return cuda_err(launch_k(k_conv3_dgrad_shift, dim3(std::min(total, g_sms)), dim3(GEMM_THREADS), C3D_SMEM, st, g),
                    "conv3 dgrad (shifted descriptors)");
}

// fc1 data gradient: dY3[b][k] = relu'(act3) * sum_j dh1[b][j] W4[j][k] (W4 as MN-major B)
int tma_fc1_dgrad(const pq_net &th, const bf16 *dh1_bf, const bf16 *act3, bf16 *dY3, int n, cudaStream_t st) {
    static thread_local TmaGemm<EpiMask> g;
    memset(&g, 0, sizeof(g));
    if (int rc = map2(&g.a[0], dh1_bf, n, 512, 512, "dh1")) return rc;
    if (int rc = map2(&g.b[0], (const bf16 *)th.shadow + S_W4, 512, 3136, 3136, "W4")) return rc;
    g.ep[0] = EpiMask{dY3, act3, n, 3136, 3136};
    g.kindA = OP_K2, g.kindB = OP_M2, g.boxesA = 2, g.boxesB = 1, g.n = n;
    g.mtiles = (n + 127) / 128, g.ntiles = 49, g.splits = 1, g.groups = 1, g.kc = 8, g.nk = 8;
    return launch_tma<64, false, true>(g, st, "fc1 dgrad (TMA)");
}

// conv3 data gradient: dY2 = relu'(act2) * transposed conv3(dY3) (im2col window, pad 2)
int tma_conv3_dgrad(const pq_net &th, const bf16 *dY3, const bf16 *act2, bf16 *dY2, int n, cudaStream_t st,
                    bf16 *dY2p, bf16 *dY2q) {
    if (dY2p) {  // also onto the padded 11 x 11 grid of the shifted conv2 data gradient
        static thread_local TmaGemm<EpiMaskPad> g;
        memset(&g, 0, sizeof(g));
        if (int rc = map_im2col(&g.a[0], dY3, n, 7, 7, -2, 0, 128, "dY3")) return rc;
        const uint64_t dims[3] = {64, 9, 64}, strd[2] = {64, 576};
        if (int rc = make_map(&g.b[0], (const bf16 *)th.shadow + S_W3, 3, dims, strd, "W3 view")) return rc;
        g.ep[0] = EpiMaskPad{EpiMask{dY2, act2, n * 81, 64, 64}, dY2p, FastDiv(81), FastDiv(9), dY2q};
        g.kindA = OP_IT3, g.kindB = OP_W3V, g.boxesA = 2, g.boxesB = 1, g.n = n, g.b_is_weight = 1;
        g.mtiles = (n * 81 + 127) / 128, g.ntiles = 1, g.splits = 1, g.groups = 1, g.kc = 9, g.nk = 9;
        return launch_tma<64, false, true>(g, st, "conv3 dgrad (TMA, padded copy)");
    }
    static thread_local TmaGemm<EpiMask> g;
    memset(&g, 0, sizeof(g));
    if (int rc = map_im2col(&g.a[0], dY3, n, 7, 7, -2, 0, 128, "dY3")) return rc;
    const uint64_t dims[3] = {64, 9, 64}, strd[2] = {64, 576};
    if (int rc = make_map(&g.b[0], (const bf16 *)th.shadow + S_W3, 3, dims, strd, "W3 view")) return rc;
    g.ep[0] = EpiMask{dY2, act2, n * 81, 64, 64};
    g.kindA = OP_IT3, g.kindB = OP_W3V, g.boxesA = 2, g.boxesB = 1, g.n = n, g.b_is_weight = 1;
    g.mtiles = (n * 81 + 127) / 128, g.ntiles = 1, g.splits = 1, g.groups = 1, g.kc = 9, g.nk = 9;
    return launch_tma<64, false, true>(g, st, "conv3 dgrad (TMA)");
}

// conv3 weight gradient: part3[s][o][k] = sum over split s of im2col(act2)[m][k] dY3[m][o];
// k = 576 is the bias row (ones tile)
int tma_conv3_wgrad(const bf16 *act2, const bf16 *dY3, float *part3, int kc, int splits, int n, cudaStream_t st) {
    static thread_local TmaGemm<EpiF32T> g;
    memset(&g, 0, sizeof(g));
    bf16 *ones = ones_tile(st);
    if (!ones) return set_err("ones tile allocation failed");
    if (int rc = map_im2col(&g.a[0], act2, n, 9, 9, 0, -2, 64, "act2 wgrad")) return rc;
    if (int rc = map2(&g.b[0], dY3, (uint64_t)n * 49, 64, 64, "dY3")) return rc;
    if (int rc = map2(&g.aux, ones, 64, 64, 64, "ones")) return rc;
    g.ep[0] = EpiF32T{part3, 577, 64, 577, (size_t)64 * 577};
    g.kindA = OP_IW3, g.kindB = OP_M2, g.boxesA = 2, g.boxesB = 1, g.n = n;
    g.mtiles = 5, g.ntiles = 1, g.splits = splits, g.groups = 1, g.kc = kc, g.nk = (n * 49 + 63) / 64;
    return launch_tma<64, true, true>(g, st, "conv3 wgrad (TMA)");
}

// conv2 data gradient per input-parity class: dY1 = relu'(act1) * transposed conv2(dY2)
int tma_conv2_dgrad(const pq_net &th, const bf16 *dY2, const bf16 *act1, bf16 *dY1, int n, cudaStream_t st,
                    int pad21) {
    static thread_local TmaGemm<EpiMaskP> g;
    memset(&g, 0, sizeof(g));
    const int tpc = (n * 100 + 127) / 128;
    if (int rc = map_im2col(&g.a[0], dY2, n, 9, 9, -1, 0, 128, "dY2")) return rc;
    const uint64_t dims[4] = {32, 4, 4, 64}, strd[3] = {32, 128, 512};
    if (int rc = make_map(&g.b[0], (const bf16 *)th.shadow + S_W2, 4, dims, strd, "W2 view")) return rc;
    g.ep[0] = epi_mask_p(dY1, act1, n, 10, 10, 32, tpc, pad21);
    g.kindA = OP_IT2, g.kindB = OP_W2V, g.boxesA = 2, g.boxesB = 1, g.n = n, g.tpc = tpc, g.b_is_weight = 1;
    g.mtiles = 4 * tpc, g.ntiles = 1, g.splits = 1, g.groups = 1, g.kc = 4, g.nk = 4;
    return launch_tma<64, false, true>(g, st, "conv2 dgrad (TMA)");
}

// ---- conv2 data gradient by row-shifted descriptors
// The stride-2 transposed conv splits into the 4 parity classes (py, px) of the 20 x 20
// input: dY1(2y+py, 2x+px) = relu'(act1) * sum_{ty,tx} dY2(y-ty, x-tx) W2[py+2ty][px+2tx].
// On the zero-padded 11 x 11 grid dY2p (dY2 at (y+1, x+1), written by conv3's data
// gradient) GEMM row r = (s, y, x) of an 11 x 11 grid (y, x = 10 discarded) reads row
// r + 11 (1 - ty) + (1 - tx) for every class, so one TMA box of 144 rows feeds all 4 taps
// x 4 classes (16 resident MN-major W2 tiles); four 64-column accumulators per tile,
// double-buffered (all 512 TMEM columns).  Same MMA order per class as the im2col
// kernel, so dY1 is bit-identical.
constexpr int C2D_ROWS = 144, C2D_BOX = C2D_ROWS * 128, C2D_STAGES = 4, C2D_W = 64 * 128;
constexpr int C2D_SMEM = 1024 + 16 * C2D_W + C2D_STAGES * C2D_BOX;
struct C2DArgs {
    CUtensorMap a, w;  // dY2p pixel rows [n*121][64]; W2 view {c1, kw, kh, c2}
    bf16 *out;         // dY1 (dense 20 x 20, or the padded 21 x 21 grid when pad21)
    const bf16 *mask;  // act1 (dense), or its 2x2 space-to-depth copy when mask_s2
    int n, pad21, mask_s2;
};

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_conv2_dgrad_shift(const __grid_constant__ C2DArgs g) {
    TlProbe tp;
    constexpr uint32_t IDESC = idesc_bf16(64, false, true);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[C2D_STAGES], empty[C2D_STAGES], accf[2], acce[2], wbar;
    __shared__ uint32_t tmem_base_s;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(smem), ring_s = w_s + 16 * C2D_W;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < C2D_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 4);
        }
        mbar_init(&wbar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&tmem_base_s);
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.w) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int total = (g.n * 121 + 127) / 128;
    if (tid == 0) {  // W2 (two launches back) before the dependency wait: tile (class, tap)
        mbar_expect_tx(&wbar, 16u * C2D_W);
        for (int cls = 0; cls < 4; ++cls)
            for (int tap = 0; tap < 4; ++tap) {
                const int kh = (cls >> 1) + 2 * (tap >> 1), kw = (cls & 1) + 2 * (tap & 1);
                tma_load_4d(w_s + (cls * 4 + tap) * C2D_W, &g.w, &wbar, 0, kw, kh, 0);
            }
    }
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t s = q % C2D_STAGES;
                if (q >= C2D_STAGES) mbar_wait(&empty[s], ((q / C2D_STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], (uint32_t)C2D_BOX);
                tma_load_2d(ring_s + s * C2D_BOX, &g.a, &full[s], 0, t * 128);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            mbar_wait(&wbar, 0);
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t buf = q & 1, s = q % C2D_STAGES;
                if (q >= 2) mbar_wait(&acce[buf], ((q >> 1) - 1) & 1);
                mbar_wait(&full[s], (q / C2D_STAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = ring_s + s * C2D_BOX;
#pragma unroll 1
                for (int cls = 0; cls < 4; ++cls) {
                    const uint32_t acc = tmem + buf * 256 + cls * 64;
#pragma unroll
                    for (int tap = 0; tap < 4; ++tap) {
                        const uint32_t shift = (uint32_t)((1 - (tap >> 1)) * 11 + (1 - (tap & 1))) * 128;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint64_t ad = desc_sw128(a0 + shift + j * 32, 0);
                            const uint64_t bd = desc_sw128(w_s + (cls * 4 + tap) * C2D_W + j * 2048, 8192);
                            umma_bf16(acc, ad, bd, IDESC, (tap > 0 || j > 0) ? 1u : 0u);
                        }
                    }
                }
                umma_commit(&empty[s]);
                umma_commit(&accf[buf]);
            }
        }
    } else if (warp >= 4) {  // epilogue
        const int wq = warp - 4;
        uint32_t q = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
            const uint32_t buf = q & 1;
            mbar_wait(&accf[buf], (q >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            const int r = t * 128 + wq * 32 + lane, smp = r / 121, p = r - smp * 121, y = p / 11, x = p - y * 11;
            const bool ok = smp < g.n && y < 10 && x < 10;
#pragma unroll 1
            for (int cls = 0; cls < 4; ++cls) {
                float v[32];
                tmem_ld32(tmem + buf * 256 + cls * 64 + ((uint32_t)(wq * 32) << 16), v);
                if (ok) {
                    const int iy = 2 * y + (cls >> 1), ix = 2 * x + (cls & 1);
                    const size_t o = ((size_t)(smp * 20 + iy) * 20 + ix) * 32;
                    const size_t oo = g.pad21 ? ((size_t)(smp * 21 + iy) * 21 + ix) * 32 : o;
                    // act1 pixel (iy, ix) = s2d pixel (y, x), channels (py * 2 + px) * 32
                    const size_t om = g.mask_s2 ? ((size_t)(smp * 10 + y) * 10 + x) * 128 + cls * 32 : o;
                    store_masked32(g.out + oo, g.mask + om, v, 32);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
    tp.done('D');
}

int tma_conv2_dgrad_shift(const pq_net &th, const bf16 *dY2p, const bf16 *act1, bf16 *dY1, int n, int pad21,
                          cudaStream_t st, int mask_s2) {
    static thread_local C2DArgs g;
    memset(&g, 0, sizeof(g));
    const uint64_t ad[2] = {64, (uint64_t)n * 121}, as[1] = {64};
    if (int rc = make_map(&g.a, dY2p, 2, ad, as, "dY2 padded rows", C2D_ROWS)) return rc;
    const uint64_t dims[4] = {32, 4, 4, 64}, strd[3] = {32, 128, 512};
    if (int rc = make_map(&g.w, (const bf16 *)th.shadow + S_W2, 4, dims, strd, "W2 view")) return rc;
    g.out = dY1, g.mask = act1, g.n = n, g.pad21 = pad21, g.mask_s2 = mask_s2;
    static bool configured = false;
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_conv2_dgrad_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, C2D_SMEM));
        configured = true;
    }
    if (!g_sms) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int total = (n * 121 + 127) / 128;
    return cuda_err(launch_k(k_conv2_dgrad_shift, dim3(std::min(total, g_sms)), dim3(GEMM_THREADS), C2D_SMEM, st, g),
                    "conv2 dgrad (shifted descriptors)");
}

// Space-to-depth gather of the frame stacks: out[b][by][bx][f*16 + dy*4 + dx] =
// frame_f[4 by + dy][4 bx + dx] (0..255 exact in bf16; slot -1 = the masked zero frame),
// f < nframes; sample b's frame slots are refs[map(b) * ref_stride + ref_off + f].  conv1
// (8x8 stride 4 over 84x84) becomes a 2x2 stride-1 conv over 21x21 pixels of 16*nframes
// channels, which TMA im2col feeds (64 channels = 4 frames from channel 16 g).
__global__ void __launch_bounds__(256) k_frames_s2d(const uint8_t *ring, const int32_t *refs, const int64_t *map,
                                                    const int32_t *counter, int map_stride, int ref_stride,
                                                    int ref_off, int nframes, bf16 *out) {
    TlProbe tp;
    // Inputs (replay ring, records, the epoch's index table and the step counter) are not
    // written by the preceding launch, and `out` was last read two launches back, so the
    // gather runs before the dependency wait (overlapping the previous step's optimizer);
    // the wait precedes the trigger so the next launch's early prologue still finds
    // everything two launches back complete.
    const int b = blockIdx.x;
    __shared__ int32_t slot[8];
    if ((int)threadIdx.x < nframes) {
        const int64_t base = (map && counter) ? (int64_t)(*counter) * map_stride : 0;
        const int64_t rec = map ? map[base + b] : (int64_t)b;
        slot[threadIdx.x] = refs[rec * ref_stride + ref_off + threadIdx.x];
    }
    __syncthreads();
    bf16 *o = out + (size_t)b * 441 * nframes * 16;
    for (int e = threadIdx.x; e < 441 * nframes; e += blockDim.x) {
        const int pix = e / nframes, f = e - pix * nframes, by = pix / 21, bx = pix - by * 21;
        const int sl = slot[f];
        uint32_t w[4] = {0, 0, 0, 0};
        if (sl >= 0) {
            const uint8_t *src = ring + (size_t)sl * FRAME_BYTES + (4 * by) * 84 + 4 * bx;
#pragma unroll
            for (int dy = 0; dy < 4; ++dy) w[dy] = __ldg(reinterpret_cast<const uint32_t *>(src + dy * 84));
        }
        uint4 *d = reinterpret_cast<uint4 *>(o + (size_t)(pix * nframes + f) * 16);
        d[0] = u8x8_to_bf16(w[0], w[1]);
        d[1] = u8x8_to_bf16(w[2], w[3]);
    }
    griddep_wait();
    griddep_launch();
    tp.waited();
    tp.done('S');
}

int tma_frames_s2d(const uint8_t *ring, const int32_t *refs, const int64_t *map, const int32_t *counter,
                   int map_stride, int ref_stride, int ref_off, int nframes, int n, bf16 *out, cudaStream_t st) {
    return cuda_err(launch_k(k_frames_s2d, dim3(n), dim3(256), 0, st, ring, refs, map, counter, map_stride, ref_stride,
                             ref_off, nframes, out),
                    "frames space-to-depth");
}

// conv1 forward on the TMA engine: act1[g] = relu(im2col(s2d, channels 16 c0g..) W1p[g]^T / 255 + b1)
int tma_conv1_fwd(const pq_net *nets, const bf16 *s2d, int nframes, const int *c0, bf16 *const *act1, int groups,
                  int n, cudaStream_t st) {
    static thread_local TmaGemm<EpiBiasRelu> g;
    memset(&g, 0, sizeof(g));
    for (int q = 0; q < groups; ++q) {
        if (int rc = map_im2col(&g.a[q], s2d, n, 21, 21, 0, -1, 128, "frames s2d", nframes * 16)) return rc;
        if (int rc = map2(&g.b[q], (const bf16 *)nets[q].shadow + S_W1P, 32, 256, 256, "W1 permuted")) return rc;
        g.ep[q] = EpiBiasRelu{act1[q], nets[q].master + P_B1, n * 400, 32, 32, 1.0f / 255.0f};
    }
    g.kindA = OP_IF1, g.kindB = OP_K2, g.boxesA = 2, g.boxesB = 1, g.n = n, g.b_is_weight = 1;
    g.tpc = 0;
    g.mtiles = (n * 400 + 127) / 128, g.ntiles = 1, g.splits = 1, g.groups = groups, g.kc = 4, g.nk = 4;
    g.cls0[0] = c0[0], g.cls0[1] = groups > 1 ? c0[1] : 0;
    return launch_tma<64, false, false>(g, st, "conv1 forward (TMA)");
}

// bias + ReLU of 32 accumulator columns (scale folded in) -> 32 bf16 at dst (and dst2):
// EpiBiasRelu's arithmetic with the biases from shared memory
PQ_DEV void bias_relu_store32(const float *v, const float *bias, float scale, bf16 *dst, bf16 *dst2) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        float y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float t = v[j + e] * scale + bias[j + e];
            y[e] = t > 0.f ? t : 0.f;
        }
        const uint4 pk = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]),
                                    pack_bf16(y[6], y[7]));
        *reinterpret_cast<uint4 *>(dst + j) = pk;
        if (dst2) *reinterpret_cast<uint4 *>(dst2 + j) = pk;
    }
}

// ---- conv1 forward as four row-shifted GEMMs over the space-to-depth stacks
// On the 21 x 21 grid of s2d pixels conv1 (8x8 / 4 over 84 x 84) is a 2 x 2 stride-1
// conv.  Computed for all 21 x 21 base pixels of a sample (outputs with y or x = 20 are
// discarded), tap (ty, tx) of GEMM row r reads s2d row r + 21 ty + tx of the same
// sample, so one TMA box of 152 rows x 64 channels feeds all four taps through UMMA
// descriptors starting 0, 1, 21 and 22 rows into it -- the SW128 swizzle is a function
// of the shared-memory address, so any 128-byte row is a valid operand start
// (scripts/desc_probe.cu) -- instead of four im2col loads (4x less L2 -> SM traffic).
// The online (channels 0..63) and target (16..79) networks share the box; the target's
// last K step (channels 64..79) comes from a second box at channel 64.  Same MMA order
// (tap, 16-channel step) as the im2col kernels, so the outputs are bit-identical.
constexpr int C1_ROWS = 152, C1_BOX = C1_ROWS * 128, C1_STAGES = 4, C1_W = 32 * 128;
constexpr int C1_SMEM = 1024 + 2 * 4 * C1_W + C1_STAGES * 2 * C1_BOX;
struct C1Args {
    CUtensorMap a, w[2];
    EpiBiasRelu ep[2];
    bf16 *act1s2[2];  // optional copy of act1 as [n][10][10][128] (2x2 space-to-depth) for k_conv2_shift
    int n, groups, coff[2];  // channel offset of group g in the s2d pixel row
    int a_early, w_early;    // operands not written by the preceding launch: load before the wait
};

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_conv1_shift(const __grid_constant__ C1Args g) {
    TlProbe tp;
    constexpr uint32_t IDESC = idesc_bf16(32, false, false);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[C1_STAGES], empty[C1_STAGES], accf[2], acce[2], wbar;
    __shared__ uint32_t tmem_base_s;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(smem), ring_s = w_s + 2 * 4 * C1_W;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < C1_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 4);  // one arrival per epilogue warp
        }
        mbar_init(&wbar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<128>(&tmem_base_s);
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a) : "memory");
        for (int q = 0; q < g.groups; ++q) asm volatile("prefetch.tensormap [%0];" ::"l"(&g.w[q]) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int total = (g.n * 441 + 127) / 128;
    const int nbox = g.coff[g.groups - 1] > 0 ? 2 : 1;
    auto load_w = [&] {
        mbar_expect_tx(&wbar, (uint32_t)(g.groups * 4 * C1_W));
        for (int q = 0; q < g.groups; ++q)
            for (int t = 0; t < 4; ++t) tma_load_2d(w_s + (q * 4 + t) * C1_W, &g.w[q], &wbar, t * 64, 0);
    };
    auto load_a = [&](uint32_t q, int t) {
        const uint32_t s = q % C1_STAGES, dst = ring_s + s * 2 * C1_BOX;
        mbar_expect_tx(&full[s], (uint32_t)(nbox * C1_BOX));
        tma_load_2d(dst, &g.a, &full[s], 0, t * 128);
        if (nbox > 1) tma_load_2d(dst + C1_BOX, &g.a, &full[s], 64, t * 128);
    };
    int pre = 0;
    if (tid == 0) {
        if (g.w_early) load_w();
        if (g.a_early)
            for (int t = blockIdx.x; t < total && pre < C1_STAGES; t += gridDim.x, ++pre) load_a(pre, t);
    }
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer
            if (!g.w_early) load_w();
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                if ((int)q < pre) continue;
                if (q >= C1_STAGES) mbar_wait(&empty[q % C1_STAGES], ((q / C1_STAGES) - 1) & 1);
                load_a(q, t);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            mbar_wait(&wbar, 0);
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t buf = q & 1, s = q % C1_STAGES;
                if (q >= 2) mbar_wait(&acce[buf], ((q >> 1) - 1) & 1);
                mbar_wait(&full[s], (q / C1_STAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = ring_s + s * 2 * C1_BOX;
                for (int gg = 0; gg < g.groups; ++gg) {
                    const uint32_t acc = tmem + buf * 64 + gg * 32;
#pragma unroll
                    for (int tap = 0; tap < 4; ++tap) {
                        const uint32_t shift = (uint32_t)((tap >> 1) * 21 + (tap & 1)) * 128;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int ch = g.coff[gg] + 16 * j;
                            const uint64_t ad = desc_sw128(a0 + (ch >> 6) * C1_BOX + shift + (ch & 63) * 2, 0);
                            const uint64_t bd = desc_sw128(w_s + (gg * 4 + tap) * C1_W + j * 32, 0);
                            umma_bf16(acc, ad, bd, IDESC, (tap > 0 || j > 0) ? 1u : 0u);
                        }
                    }
                }
                umma_commit(&empty[s]);
                umma_commit(&accf[buf]);
            }
        }
    } else if (warp >= 4) {  // epilogue: TMEM lane quadrant = warp % 4
        const int wq = warp - 4;
        __shared__ float s_bias[2][32];  // conv1 biases (after the wait: the update is upstream)
        if (wq == 0)
            for (int gg = 0; gg < g.groups; ++gg) s_bias[gg][lane] = g.ep[gg].bias[lane];
        named_bar_sync(1, 128);
        uint32_t q = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
            const uint32_t buf = q & 1;
            mbar_wait(&accf[buf], (q >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            float v[2][32];
            const uint32_t trow = tmem + buf * 64 + ((uint32_t)(wq * 32) << 16);
            tmem_ld32(trow, v[0]);
            if (g.groups > 1) tmem_ld32(trow + 32, v[1]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[buf]);
            const int r = t * 128 + wq * 32 + lane, smp = r / 441, p = r - smp * 441, y = p / 21, x = p - y * 21;
            if (smp < g.n && y < 20 && x < 20) {
                const int m = smp * 400 + y * 20 + x;
                // the 2x2 space-to-depth copy: pixel (y, x) -> (y/2, x/2), channels ((y&1)*2 + (x&1))*32
                const size_t o2 = ((size_t)(smp * 10 + (y >> 1)) * 10 + (x >> 1)) * 128 + ((y & 1) * 2 + (x & 1)) * 32;
#pragma unroll
                for (int gg = 0; gg < 2; ++gg) {
                    if (gg >= g.groups) break;
                    const EpiBiasRelu &e = g.ep[gg];
                    bf16 *d1 = e.out ? e.out + (size_t)m * e.ld : nullptr;  // dense act1 (absent with the copy)
                    bf16 *d2 = g.act1s2[gg] ? g.act1s2[gg] + o2 : nullptr;   // 2x2 space-to-depth copy
                    bias_relu_store32(v[gg], s_bias[gg], e.scale, d1 ? d1 : d2, d1 ? d2 : nullptr);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
    tp.done('1');
}

// conv1 forward by row-shifted descriptors (k_conv1_shift): groups online / target over
// channel offsets c0[g] of the s2d stacks (16 * nframes channels per pixel)
int tma_conv1_shift(const pq_net *nets, const bf16 *s2d, int nframes, const int *c0, bf16 *const *act1,
                    int groups, int n, int a_early, int w_early, cudaStream_t st, bf16 *const *act1s2) {
    static thread_local C1Args g;
    memset(&g, 0, sizeof(g));
    for (int q = 0; q < groups && act1s2; ++q) g.act1s2[q] = act1s2[q];
    const uint64_t ad[2] = {(uint64_t)nframes * 16, (uint64_t)n * 441}, as[1] = {(uint64_t)nframes * 16};
    if (int rc = make_map(&g.a, s2d, 2, ad, as, "s2d pixel rows", C1_ROWS)) return rc;
    for (int q = 0; q < groups; ++q) {
        const uint64_t wd[2] = {256, 32}, ws[1] = {256};
        if (int rc = make_map(&g.w[q], (const bf16 *)nets[q].shadow + S_W1P, 2, wd, ws, "W1 permuted", 32))
            return rc;
        // with the space-to-depth copy the dense act1 has no reader (conv2 forward / weight
        // gradient read the copy, conv2's data gradient takes its ReLU mask from it)
        g.ep[q] = EpiBiasRelu{act1s2 ? nullptr : act1[q], nets[q].master + P_B1, n * 400, 32, 32, 1.0f / 255.0f};
        g.coff[q] = c0[q];
    }
    if (groups > 1 && (c0[1] + 64 > nframes * 16 || c0[0] != 0)) return set_err("conv1 shift: channel window");
    g.n = n, g.groups = groups, g.a_early = a_early, g.w_early = w_early;
    static bool configured = false;
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_conv1_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, C1_SMEM));
        configured = true;
    }
    if (!g_sms) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int total = (n * 441 + 127) / 128;
    return cuda_err(launch_k(k_conv1_shift, dim3(std::min(total, g_sms)), dim3(GEMM_THREADS), C1_SMEM, st, g),
                    "conv1 forward (shifted descriptors)");
}

// ---- conv2 / conv3 forward by row-shifted descriptors
// conv2: act1s2[s][Y][X][(dy*2 + dx)*32 + c] = act1[s][2Y+dy][2X+dx][c] (written by
// k_conv1_shift) turns conv2 (4x4 / 2 over 20 x 20 x 32) into a 2 x 2 stride-1 conv over
// 10 x 10 x 128: GEMM row r = (s, Y, X) of the 10 x 10 grid (Y, X = 9 discarded), tap
// (ty, tx) reads row r + 10 ty + tx; one TMA box of 144 rows per 64-channel half
// (dy = 0 / 1).  conv3 (3x3 / 1 over 9 x 9 x 64): the 7 x 7 outputs on the 9 x 9 grid of
// act2 itself, tap (ky, kx) reads row r + 9 ky + kx; one box of 148 rows.  The MMAs run in
// the K order of the im2col kernels (K chunk c of W is its plain 64-column block: conv2
// ky = c >> 1, kx pair c & 1; conv3 tap c), so the activations are bit-identical.
template <int CV>
struct ConvShift {
    static constexpr int GW = CV == 2 ? 10 : 9;    // grid width (rows per grid row)
    static constexpr int RPS = GW * GW;            // grid rows per sample
    static constexpr int OW = CV == 2 ? 9 : 7;     // valid output width
    static constexpr int NCH = CV == 2 ? 8 : 9;    // 64-wide K chunks
    static constexpr int NBOX = CV == 2 ? 2 : 1;   // 64-channel boxes per pixel row
    static constexpr int ROWS = CV == 2 ? 144 : 152;
    static constexpr int BOX = ROWS * 128, W = 64 * 128, STAGES = 2;
    static constexpr int SMEM = 1024 + 2 * NCH * W + STAGES * NBOX * BOX;
    PQ_HD static int box_of(int c) { return CV == 2 ? ((c >> 1) & 1) : 0; }
    PQ_HD static int shift_of(int c) { return CV == 2 ? ((c >> 2) * 10 + (c & 1)) : ((c / 3) * 9 + c % 3); }
};
struct CSArgs {
    CUtensorMap a[2], w[2];  // input pixel rows [n*RPS][64*NBOX]; W [64][64*NCH]
    EpiBiasRelu ep[2];       // output [n*OW*OW][64]
    int n, groups;
};

template <int CV>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_conv_shift(const __grid_constant__ CSArgs g) {
    using C = ConvShift<CV>;
    constexpr uint32_t IDESC = idesc_bf16(64, false, false);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[C::STAGES], empty[C::STAGES], accf[2], acce[2], wbar;
    __shared__ uint32_t tmem_base_s;
    TlProbe tp;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(smem), ring_s = w_s + 2 * C::NCH * C::W;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 4);
        }
        mbar_init(&wbar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<128>(&tmem_base_s);
    if (tid == 32)
        for (int q = 0; q < g.groups; ++q) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a[q]) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&g.w[q]) : "memory");
        }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int mt = (g.n * C::RPS + 127) / 128, total = mt * g.groups;
    if (tid == 0) {  // weights (updated two or more launches back) before the dependency wait
        mbar_expect_tx(&wbar, (uint32_t)(g.groups * C::NCH * C::W));
        for (int q = 0; q < g.groups; ++q)
            for (int c = 0; c < C::NCH; ++c) tma_load_2d(w_s + (q * C::NCH + c) * C::W, &g.w[q], &wbar, c * 64, 0);
    }
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer: tile t = (m-tile t / groups, group t % groups)
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t s = q % C::STAGES, dst = ring_s + s * C::NBOX * C::BOX;
                const int grp = t % g.groups, m = t / g.groups;
                if (q >= C::STAGES) mbar_wait(&empty[s], ((q / C::STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], (uint32_t)(C::NBOX * C::BOX));
                for (int b = 0; b < C::NBOX; ++b) tma_load_2d(dst + b * C::BOX, &g.a[grp], &full[s], b * 64, m * 128);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            mbar_wait(&wbar, 0);
            uint32_t q = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
                const uint32_t buf = q & 1, s = q % C::STAGES;
                const int grp = t % g.groups;
                if (q >= 2) mbar_wait(&acce[buf], ((q >> 1) - 1) & 1);
                mbar_wait(&full[s], (q / C::STAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = ring_s + s * C::NBOX * C::BOX, acc = tmem + buf * 64;
#pragma unroll
                for (int c = 0; c < C::NCH; ++c) {
                    const uint32_t abase = a0 + C::box_of(c) * C::BOX + (uint32_t)C::shift_of(c) * 128;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t ad = desc_sw128(abase + j * 32, 0);
                        const uint64_t bd = desc_sw128(w_s + (grp * C::NCH + c) * C::W + j * 32, 0);
                        umma_bf16(acc, ad, bd, IDESC, (c > 0 || j > 0) ? 1u : 0u);
                    }
                }
                umma_commit(&empty[s]);
                umma_commit(&accf[buf]);
            }
        }
    } else if (warp >= 4) {  // epilogue
        const int wq = warp - 4;
        __shared__ float s_bias[2][64];
        if (wq < g.groups)
            for (int c = lane; c < 64; c += 32) s_bias[wq][c] = g.ep[wq].bias[c];
        named_bar_sync(1, 128);
        uint32_t q = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++q) {
            const uint32_t buf = q & 1;
            const int grp = t % g.groups, m = t / g.groups;
            mbar_wait(&accf[buf], (q >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            float v[2][32];
            const uint32_t trow = tmem + buf * 64 + ((uint32_t)(wq * 32) << 16);
            tmem_ld32(trow, v[0]);
            tmem_ld32(trow + 32, v[1]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[buf]);
            const int r = m * 128 + wq * 32 + lane, smp = r / C::RPS, p = r - smp * C::RPS, y = p / C::GW,
                      x = p - y * C::GW;
            if (smp < g.n && y < C::OW && x < C::OW) {
                const int o = (smp * C::OW + y) * C::OW + x;
                bf16 *dst = g.ep[grp].out + (size_t)o * 64;
                bias_relu_store32(v[0], s_bias[grp], 1.0f, dst, nullptr);
                bias_relu_store32(v[1], s_bias[grp] + 32, 1.0f, dst + 32, nullptr);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
    tp.done(CV == 2 ? '2' : '3');
}

template <int CV>
static int launch_conv_shift(const pq_net *nets, bf16 *const *in, bf16 *const *out, int groups, int n, cudaStream_t st) {
    using C = ConvShift<CV>;
    static thread_local CSArgs g;
    memset(&g, 0, sizeof(g));
    const int64_t wofs = CV == 2 ? S_W2 : S_W3, bofs = CV == 2 ? P_B2 : P_B3;
    for (int q = 0; q < groups; ++q) {
        const uint64_t ad[2] = {(uint64_t)64 * C::NBOX, (uint64_t)n * C::RPS}, as[1] = {(uint64_t)64 * C::NBOX};
        if (int rc = make_map(&g.a[q], in[q], 2, ad, as, "conv input pixel rows", C::ROWS)) return rc;
        if (int rc = map2(&g.w[q], (const bf16 *)nets[q].shadow + wofs, 64, 64 * C::NCH, 64 * C::NCH, "conv W"))
            return rc;
        g.ep[q] = EpiBiasRelu{out[q], nets[q].master + bofs, n * C::OW * C::OW, 64, 64, 1.0f};
    }
    g.n = n, g.groups = groups;
    static bool configured = false;
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_conv_shift<CV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        configured = true;
    }
    if (!g_sms) {
        int dev = 0;
        PQ_CUDA_TRY(cudaGetDevice(&dev));
        PQ_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int total = ((n * C::RPS + 127) / 128) * groups;
    return cuda_err(launch_k(k_conv_shift<CV>, dim3(std::min(total, g_sms)), dim3(GEMM_THREADS), C::SMEM, st, g),
                    CV == 2 ? "conv2 forward (shifted descriptors)" : "conv3 forward (shifted descriptors)");
}
int tma_conv2_shift(const pq_net *nets, bf16 *const *act1s2, bf16 *const *act2, int groups, int n, cudaStream_t st) {
    return launch_conv_shift<2>(nets, act1s2, act2, groups, n, st);
}
int tma_conv3_shift(const pq_net *nets, bf16 *const *act2, bf16 *const *act3, int groups, int n, cudaStream_t st) {
    return launch_conv_shift<3>(nets, act2, act3, groups, n, st);
}

// ---- conv2 weight gradient by row-shifted descriptors (the transpose of k_conv2_shift)
// part2[split][c2][k] (k = (ky*4 + kx)*32 + c, the im2col order; k = 512 the bias row) =
// sum over the split's rows r of the 10 x 10 grid of act1s2[r + 10 ty + tx][ch] dY2q[r][c2]
// with dY2q = conv3's data gradient on that grid (zero rows at y or x = 9).  For tap
// (ty, tx) the 128 channels of a space-to-depth pixel are the two contiguous 64-wide K
// blocks ky = 2 ty + dy, kx = 2 tx .. 2 tx + 1: M tile = one tap, its two MN-major atoms
// are the two 64-channel boxes at the same row shift (LBO = box distance); M tile 4 = a
// ones column (bias row).  One CTA per split runs all five M tiles (320 TMEM columns).
constexpr int W2S_ROWS = 80, W2S_ABOX = W2S_ROWS * 128, W2S_BBOX = 64 * 128, W2S_STAGES = 5;
constexpr int W2S_SLOT = 2 * W2S_ABOX + W2S_BBOX;  // 28 KB, 1024-aligned
constexpr int W2S_SMEM = 1024 + 2 * 8192 + W2S_STAGES * W2S_SLOT;
struct W2SArgs {
    CUtensorMap a, b;  // act1s2 pixel rows [n*100][128]; dY2q [n*100][64]
    EpiF32T ep;        // part2[split][64][513]
    int nk, kc;
};

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_conv2_wgrad_shift(const __grid_constant__ W2SArgs g) {
    constexpr uint32_t IDESC = idesc_bf16(64, true, true);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[W2S_STAGES], empty[W2S_STAGES], accf;
    __shared__ uint32_t tmem_base_s;
    TlProbe tp;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t ones_s = smem_u32(smem), ring_s = ones_s + 2 * 8192;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 2 * 8192 / 16; i += blockDim.x) {  // ones operand: M index 0 = 1
        const int atom = i >> 9, k = (i >> 3) & 63, c8 = i & 7;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (atom == 0 && c8 == 0) val.x = 0x3F80u;
        *reinterpret_cast<uint4 *>(smem + atom * 8192 + mnmaj_off(k, c8) % 8192) = val;
    }
    if (tid == 0) {
        for (int s = 0; s < W2S_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&accf, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&tmem_base_s);
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.b) : "memory");
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int split = blockIdx.x, kb0 = split * g.kc, kb1 = min(g.nk, kb0 + g.kc);
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer
            uint32_t q = 0;
            for (int kb = kb0; kb < kb1; ++kb, ++q) {
                const uint32_t s = q % W2S_STAGES, dst = ring_s + s * W2S_SLOT;
                if (q >= W2S_STAGES) mbar_wait(&empty[s], ((q / W2S_STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], (uint32_t)W2S_SLOT);
                tma_load_2d(dst, &g.a, &full[s], 0, kb * 64);
                tma_load_2d(dst + W2S_ABOX, &g.a, &full[s], 64, kb * 64);
                tma_load_2d(dst + 2 * W2S_ABOX, &g.b, &full[s], 0, kb * 64);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer: five 128 x 64 accumulators
            uint32_t q = 0;
            for (int kb = kb0; kb < kb1; ++kb, ++q) {
                const uint32_t s = q % W2S_STAGES;
                mbar_wait(&full[s], (q / W2S_STAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = ring_s + s * W2S_SLOT, b0 = a0 + 2 * W2S_ABOX;
#pragma unroll
                for (int j = 0; j < 4; ++j) {  // K steps of 16 rows (2048 B)
                    const uint32_t acc_on = (kb > kb0 || j > 0) ? 1u : 0u;
                    const uint64_t bd = desc_sw128(b0 + j * 2048, 8192);
#pragma unroll
                    for (int tap = 0; tap < 4; ++tap) {
                        const uint32_t shift = (uint32_t)((tap >> 1) * 10 + (tap & 1)) * 128;
                        umma_bf16(tmem + tap * 64, desc_sw128(a0 + shift + j * 2048, W2S_ABOX), bd, IDESC, acc_on);
                    }
                    umma_bf16(tmem + 256, desc_sw128(ones_s + j * 2048, 8192), bd, IDESC, acc_on);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(&accf);
        }
    } else if (warp >= 4) {  // epilogue: M row i of tap tile -> k
        const int wq = warp - 4;
        mbar_wait(&accf, 0);
        __syncwarp();
        tc_fence_after();
#pragma unroll 1
        for (int mt = 0; mt < 5; ++mt) {
            const int i = wq * 32 + lane;
            int k;
            if (mt < 4) {
                const int ty = mt >> 1, tx = mt & 1, dy = i >> 6;
                k = ((2 * ty + dy) * 4 + 2 * tx) * 32 + (i & 63);
            } else {
                k = i == 0 ? 512 : -1;
            }
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                float v[32];
                if (kb1 > kb0) {
                    tmem_ld32(tmem + mt * 64 + h * 32 + ((uint32_t)(wq * 32) << 16), v);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
                if (k >= 0) g.ep.apply(k, h * 32, v, 32, split);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
    tp.done('V');
}

int tma_conv2_wgrad_shift(const bf16 *act1s2, const bf16 *dY2q, float *part2, int kc, int splits, int n,
                          cudaStream_t st) {
    static thread_local W2SArgs g;
    memset(&g, 0, sizeof(g));
    const uint64_t ad[2] = {128, (uint64_t)n * 100}, as[1] = {128};
    if (int rc = make_map(&g.a, act1s2, 2, ad, as, "act1 s2d rows (wgrad)", W2S_ROWS)) return rc;
    if (int rc = map2(&g.b, dY2q, (uint64_t)n * 100, 64, 64, "dY2 10x10")) return rc;
    g.ep = EpiF32T{part2, 513, 64, 513, (size_t)64 * 513};
    g.nk = (n * 100 + 63) / 64;
    g.kc = kc;
    const int grid = (g.nk + kc - 1) / kc;
    if (grid != splits) return set_err("conv2 wgrad shift: split count mismatch");
    static bool configured = false;
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_conv2_wgrad_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, W2S_SMEM));
        configured = true;
    }
    return cuda_err(launch_k(k_conv2_wgrad_shift, dim3(grid), dim3(GEMM_THREADS), W2S_SMEM, st, g),
                    "conv2 wgrad (shifted descriptors)");
}

// ---- conv1 weight gradient by row-shifted descriptors (the transpose of k_conv1_shift)
// part1[split][k'][o] = sum over the split's rows r of the padded 21 x 21 grid of
// s2d[r + 21 ty + tx][c] dY1p[r][o] (k' = tap * 64 + c, tap = (ty, tx)), row 256 = the
// bias gradient sum_r dY1p[r][o].  dY1p holds conv2's data gradient on the same padded
// grid (zero rows at y or x = 20, written by tma_conv2_dgrad(pad21)), so one TMA box of
// 88 s2d rows per 64-row K chunk feeds all four taps as MN-major operands: M tile 0 =
// taps (0,0), (0,1) (rows +0 / +1: start +0, LBO 128 B), M tile 1 = taps (1,0), (1,1)
// (start +21 rows, LBO 128 B), M tile 2 = a ones column (bias row).  One CTA per split
// runs all three M tiles from the same operands.
constexpr int W1S_ROWS = 88, W1S_ABOX = W1S_ROWS * 128, W1S_BBOX = 64 * 128, W1S_STAGES = 6;
constexpr int W1S_SLOT = ((W1S_ABOX + W1S_BBOX + 1023) / 1024) * 1024;
constexpr int W1S_SMEM = 1024 + 2 * 8192 + W1S_STAGES * W1S_SLOT;
struct W1SArgs {
    CUtensorMap a, b;  // s2d pixel rows [n*441][16*nframes]; dY1p [n*441][32]
    EpiF32T ep;        // part1[split][257][32]
    int nk, kc;        // 64-row K chunks in all, per split
};

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_conv1_wgrad_shift(const __grid_constant__ W1SArgs g) {
    TlProbe tp;
    constexpr uint32_t IDESC = idesc_bf16(64, true, true);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[W1S_STAGES], empty[W1S_STAGES], accf;
    __shared__ uint32_t tmem_base_s;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t ones_s = smem_u32(smem), ring_s = ones_s + 2 * 8192;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ones operand (MN-major, 64 K rows x 128 B per M atom, two atoms): M index 0 = 1
    for (int i = tid; i < 2 * 8192 / 16; i += blockDim.x) {
        const int atom = i >> 9, k = (i >> 3) & 63, c8 = i & 7;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (atom == 0 && c8 == 0) val.x = 0x3F80u;  // bf16 1.0 at M index 0 of every K row
        *reinterpret_cast<uint4 *>(smem + atom * 8192 + mnmaj_off(k, c8) % 8192) = val;
    }
    if (tid == 0) {
        for (int s = 0; s < W1S_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&accf, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<256>(&tmem_base_s);
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&g.b) : "memory");
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const int split = blockIdx.x, kb0 = split * g.kc, kb1 = min(g.nk, kb0 + g.kc);
    // the frames (written two launches back) go out before the dependency wait
    int pre = 0;
    if (tid == 0)
        for (int kb = kb0; kb < kb1 && pre < W1S_STAGES; ++kb, ++pre) {
            mbar_expect_tx(&full[pre], (uint32_t)(W1S_ABOX + W1S_BBOX));
            tma_load_2d(ring_s + pre * W1S_SLOT, &g.a, &full[pre], 0, kb * 64);
        }
    griddep_wait();
    griddep_launch();
    tp.waited();
    if (warp == 0) {
        if (lane == 0) {  // producer
            uint32_t q = 0;
            for (int kb = kb0; kb < kb1; ++kb, ++q) {
                const uint32_t s = q % W1S_STAGES, dst = ring_s + s * W1S_SLOT;
                if ((int)q >= pre) {
                    if (q >= W1S_STAGES) mbar_wait(&empty[s], ((q / W1S_STAGES) - 1) & 1);
                    mbar_expect_tx(&full[s], (uint32_t)(W1S_ABOX + W1S_BBOX));
                    tma_load_2d(dst, &g.a, &full[s], 0, kb * 64);
                }
                tma_load_2d(dst + W1S_ABOX, &g.b, &full[s], 0, kb * 64);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer: three 128 x 64 accumulators
            uint32_t q = 0;
            for (int kb = kb0; kb < kb1; ++kb, ++q) {
                const uint32_t s = q % W1S_STAGES;
                mbar_wait(&full[s], (q / W1S_STAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = ring_s + s * W1S_SLOT, b0 = a0 + W1S_ABOX;
#pragma unroll
                for (int j = 0; j < 4; ++j) {  // K steps of 16 rows (2048 B)
                    const uint32_t acc_on = (kb > kb0 || j > 0) ? 1u : 0u;
                    const uint64_t bd = desc_sw128(b0 + j * 2048, 8192);
                    umma_bf16(tmem, desc_sw128(a0 + j * 2048, 128), bd, IDESC, acc_on);
                    umma_bf16(tmem + 64, desc_sw128(a0 + 21 * 128 + j * 2048, 128), bd, IDESC, acc_on);
                    umma_bf16(tmem + 128, desc_sw128(ones_s + j * 2048, 8192), bd, IDESC, acc_on);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(&accf);
        }
    } else if (warp >= 4) {  // epilogue
        const int wq = warp - 4;
        mbar_wait(&accf, 0);
        __syncwarp();
        tc_fence_after();
#pragma unroll 1
        for (int mt = 0; mt < 3; ++mt) {
            float v[32];
            const int row = mt * 128 + wq * 32 + lane;
            if (kb1 > kb0) {
                tmem_ld32(tmem + mt * 64 + ((uint32_t)(wq * 32) << 16), v);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.f;
            }
            if (mt < 2 || row == 256) g.ep.apply(row, 0, v, 32, split);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tmem);
    tp.done('W');
}

int tma_conv1_wgrad_shift(const bf16 *s2d, int nframes, const bf16 *dY1p, float *part1, int kc, int splits,
                          int n, cudaStream_t st) {
    static thread_local W1SArgs g;
    memset(&g, 0, sizeof(g));
    const uint64_t ad[2] = {(uint64_t)nframes * 16, (uint64_t)n * 441}, as[1] = {(uint64_t)nframes * 16};
    if (int rc = make_map(&g.a, s2d, 2, ad, as, "s2d pixel rows (wgrad)", W1S_ROWS)) return rc;
    if (int rc = map2(&g.b, dY1p, (uint64_t)n * 441, 32, 32, "dY1 padded")) return rc;
    g.ep = EpiF32T{part1, 257, 32, 257, (size_t)32 * 257};
    g.nk = (n * 441 + 63) / 64;
    g.kc = kc;
    const int grid = (g.nk + kc - 1) / kc;
    if (grid != splits) return set_err("conv1 wgrad shift: split count mismatch");
    static bool configured = false;
    if (!configured) {
        PQ_CUDA_TRY(cudaFuncSetAttribute(k_conv1_wgrad_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, W1S_SMEM));
        configured = true;
    }
    return cuda_err(launch_k(k_conv1_wgrad_shift, dim3(grid), dim3(GEMM_THREADS), W1S_SMEM, st, g),
                    "conv1 wgrad (shifted descriptors)");
}

// conv1 weight gradient on the TMA engine: part1[s][o][k'] over the permuted K order
// (k' = 256: bias row from the ones tile)
int tma_conv1_wgrad(const bf16 *s2d, int nframes, const bf16 *dY1, float *part1, int kc, int splits, int n,
                    cudaStream_t st) {
    static thread_local TmaGemm<EpiF32T> g;
    memset(&g, 0, sizeof(g));
    bf16 *ones = ones_tile(st);
    if (!ones) return set_err("ones tile allocation failed");
    if (int rc = map_im2col(&g.a[0], s2d, n, 21, 21, 0, -1, 64, "frames s2d wgrad", nframes * 16)) return rc;
    if (int rc = map2(&g.b[0], dY1, (uint64_t)n * 400, 32, 32, "dY1")) return rc;
    if (int rc = map2(&g.aux, ones, 64, 64, 64, "ones")) return rc;
    g.ep[0] = EpiF32T{part1, 257, 32, 257, (size_t)32 * 257};
    g.kindA = OP_IW1, g.kindB = OP_M2, g.boxesA = 2, g.boxesB = 1, g.n = n;
    g.mtiles = 3, g.ntiles = 1, g.splits = splits, g.groups = 1, g.kc = kc, g.nk = (n * 400 + 63) / 64;
    return launch_tma<64, true, true>(g, st, "conv1 wgrad (TMA)");
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

// GEMM timeline probes of this translation unit (layout of pq_timeline)
int pq_plearn_timeline(int on, unsigned long long *out, int *count) {
    if (out) {
        static Timeline h;
        PQ_CUDA_TRY(cudaMemcpyFromSymbol(&h, g_tl, sizeof(Timeline)));
        *count = h.n < 256 ? h.n : 256;
        memcpy(out, h.t, sizeof(h.t));
    }
    static Timeline z;
    memset(&z, 0, sizeof(z));
    z.on = on;
    PQ_CUDA_TRY(cudaMemcpyToSymbol(g_tl, &z, sizeof(Timeline)));
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
    static PLearnArgs a;  // large (tensor maps + schedules): not on the stack
    memset(&a, 0, sizeof(a));
    a.theta = la->theta, a.target = la->target, a.opt = la->opt;
    a.ring = la->ring, a.records = la->records, a.idx_base = la->idx_base;
    a.update_counter = la->update_counter;
    a.n = n, a.A = la->actions, a.n8 = (n + 7) & ~7, a.n_updates = n_updates;
    a.gamma = la->gamma, a.lr = la->lr, a.rho = la->rho, a.kappa = la->kappa;
    a.nonfinite = la->nonfinite, a.grad_out = la->grad_out, a.q_out = la->q_out, a.td_out = la->td_out;
    a.wsb = (bf16 *)la->ws;
    a.act1 = w.act1;
    for (int g = 0; g < 2; ++g) {
        for (int p = 0; p < 2; ++p) {
            a.act3[g][p] = w.act3[g][p], a.P1[g][p] = w.P1[g][p], a.fc1part[g][p] = w.fc1part[g][p];
        }
        a.P2[g] = w.P2[g], a.act2[g] = w.act2[g];
    }
    a.ones = w.ones;
    a.q = w.q, a.h1 = w.h1, a.dh1 = w.dh1, a.td = w.td, a.dh1_bf = w.dh1_bf, a.dh1T = w.dh1T, a.act = w.act;
    a.dY3 = w.dY3, a.dY2 = w.dY2, a.dY1 = w.dY1;
    a.part1 = w.part1, a.part2 = w.part2, a.part3 = w.part3;
    a.bar = w.bar;
    a.trace = g_trace;
    if (int rc = build_maps(a)) return rc;
    build_plans(a, G);
    PQ_CUDA_TRY(cudaMemsetAsync(w.bar, 0, sizeof(unsigned), st));
    k_plearn_ones<<<64, 256, 0, st>>>(w.P1[0][0], w.P1[0][1], w.P2[0], w.ones, n);
    PQ_CUDA_TRY(cudaGetLastError());
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
