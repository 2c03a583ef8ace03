// GPU-resident replay memory: numpy-exact index sampling, 4-frame-stack gather,
// owner-major flush and device prepopulation.
//
//   ReplayMemory.sample   replay.py:61-66  -> k_sample_indices (PCG64 + buffered Lemire,
//                                             bit-exact with Generator.integers)
//   batch stack gather    agent.py:76,:100 -> k_gather (5 unique frames in, 8 out)
//   ReplayMemory.flush    replay.py:82-93  -> k_flush (owner-major slot order)
//   ReplayMemory.prepopulate replay.py:68-80 -> k_prepop_scalar + k_gen_frames
#include <cstdio>

#include "../../include/paraq_b200.h"
#include "common.cuh"
#include "qnet.cuh"

#define PQ_CHECK(expr, where)                          \
    do {                                               \
        int _rc = pq::cuda_err((expr), (where));       \
        if (_rc) return _rc;                           \
    } while (0)

namespace pq {
int set_err(const char *msg);
int cuda_err(cudaError_t e, const char *where);

// ------------------------------------------------------------------ sampling
constexpr int SAMPLE_THREADS = 1024;
constexpr int SAMPLE_PER = 32;  // 64-bit outputs per thread per round

__device__ __forceinline__ U128 pcg_step(U128 s, U128 inc) {
    return add128(mul128(s, U128{PCG_MULT_HI, PCG_MULT_LO}), inc);
}

// Parallel restatement of numpy's sequential draw: every thread generates a
// contiguous run of 64-bit outputs by LCG jump-ahead, Lemire-accepts each 32-bit
// half (lo then hi, the has_uint32 order), and a block scan places accepted values
// in stream order.  The state after the count-th accepted draw (including the
// buffered high half) is written back exactly as numpy would leave it.
__global__ void __launch_bounds__(SAMPLE_THREADS) k_sample_indices(uint64_t *st, uint32_t n,
                                                                   int64_t count, int64_t *out) {
    __shared__ int64_t s_produced;
    __shared__ int s_warp[SAMPLE_THREADS / 32];
    __shared__ int s_total;
    __shared__ uint64_t s_fin[6];
    __shared__ int s_done;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (count <= 0) return;
    if (n <= 1) {
        for (int64_t i = tid; i < count; i += SAMPLE_THREADS) out[i] = 0;
        return;
    }
    const uint32_t threshold = (0u - n) % n;
    Pcg64 g;
    g.load(st);
    const U128 inc = g.inc;
    U128 base = g.state;
    if (tid == 0) {
        s_produced = 0;
        s_done = 0;
        for (int k = 0; k < 6; ++k) s_fin[k] = st[k];
        if (g.has32) {
            uint64_t m = (uint64_t)g.buf * n;
            s_fin[4] = 0;  // the buffered half is consumed
            if ((uint32_t)m >= threshold) {
                out[0] = (int64_t)(m >> 32);
                s_produced = 1;
            }
            if (s_produced == count) s_done = 1;
        }
    }
    __syncthreads();
    while (!s_done) {
        const int64_t produced = s_produced;
        U128 s0 = pcg_advance(base, inc, (uint64_t)tid * SAMPLE_PER);
        int cnt = 0;
        U128 s = s0;
        for (int o = 0; o < SAMPLE_PER; ++o) {
            s = pcg_step(s, inc);
            uint64_t v = pcg_output(s);
            cnt += ((uint32_t)((uint64_t)(uint32_t)v * n) >= threshold);
            cnt += ((uint32_t)((uint64_t)(uint32_t)(v >> 32) * n) >= threshold);
        }
        // block exclusive scan of cnt
        int x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int wv = lane < SAMPLE_THREADS / 32 ? s_warp[lane] : 0;
            int ws = wv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += y;
            }
            if (lane < SAMPLE_THREADS / 32) s_warp[lane] = ws - wv;
            if (lane == 31) s_total = ws;
        }
        __syncthreads();
        int64_t k = produced + s_warp[warp] + (x - cnt);
        s = s0;
        for (int o = 0; o < SAMPLE_PER; ++o) {
            s = pcg_step(s, inc);
            uint64_t v = pcg_output(s);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t u = half ? (uint32_t)(v >> 32) : (uint32_t)v;
                uint64_t m = (uint64_t)u * n;
                if ((uint32_t)m >= threshold) {
                    if (k < count) out[k] = (int64_t)(m >> 32);
                    if (k == count - 1) {
                        s_fin[0] = s.hi;
                        s_fin[1] = s.lo;
                        s_fin[4] = half ? 0 : 1;
                        s_fin[5] = (uint32_t)(v >> 32);  // numpy leaves uinteger = hi
                    }
                    ++k;
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (produced + s_total >= count) {
                s_done = 1;
            } else {
                s_produced = produced + s_total;
            }
        }
        base = pcg_advance(base, inc, (uint64_t)SAMPLE_THREADS * SAMPLE_PER);
        __syncthreads();
    }
    if (tid == 0) {
        for (int k = 0; k < 6; ++k) st[k] = s_fin[k];
    }
}

// ------------------------------------------------------------------ gather
// one block per sampled transition: read the 5 unique frames once (16 B vector
// loads), write the two 4-frame stacks (masked slots -> zeros)
__global__ void __launch_bounds__(256) k_gather(const uint8_t *ring, const int32_t *records,
                                                const int64_t *idx, uint8_t *s_out,
                                                uint8_t *s2_out, int32_t *a_out, double *r_out,
                                                uint8_t *term_out) {
    const int b = blockIdx.x;
    const int32_t *rec = records + idx[b] * REC_INTS;
    __shared__ int32_t f[REC_INTS];
    if (threadIdx.x < REC_INTS) f[threadIdx.x] = rec[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        a_out[b] = rec_action(f[5]);
        r_out[b] = rec_reward(f[6], f[7]);
        term_out[b] = (uint8_t)rec_terminal(f[5]);
    }
    constexpr int V = FRAME_BYTES / 16;  // 441
    uint4 *s4 = reinterpret_cast<uint4 *>(s_out + (size_t)b * 4 * FRAME_BYTES);
    uint4 *t4 = reinterpret_cast<uint4 *>(s2_out + (size_t)b * 4 * FRAME_BYTES);
    for (int e = threadIdx.x; e < 5 * V; e += blockDim.x) {
        int fr = e / V, off = e - fr * V;
        int slot = f[fr];
        uint4 v = slot < 0 ? make_uint4(0, 0, 0, 0)
                           : __ldg(reinterpret_cast<const uint4 *>(ring + (size_t)slot * FRAME_BYTES) + off);
        if (fr < 4) s4[fr * V + off] = v;
        if (fr > 0) t4[(fr - 1) * V + off] = v;
    }
}

// TMA variant: one elected thread per CTA moves whole 84x84 frames with bulk copies --
// cp.async.bulk global -> shared (mbarrier complete_tx) for the <= 5 unique frames of a
// transition, then 8 bulk stores shared -> global for the two stacks (masked slots store
// from a zeroed tile) -- through an NS-deep ring of 5-frame stages, so the loads of the
// next NS-1 transitions are in flight while the current one is written out.  No register
// staging, no address arithmetic per 16 bytes; persistent grid (2 CTAs per SM).
template <int NS>
__global__ void __launch_bounds__(32) k_gather_tma(const uint8_t *ring, const int32_t *records,
                                                   const int64_t *idx, int64_t B, uint8_t *s_out,
                                                   uint8_t *s2_out, int32_t *a_out, double *r_out,
                                                   uint8_t *term_out) {
    extern __shared__ __align__(128) uint8_t gsm[];
    __shared__ uint64_t bars[NS];
    uint8_t *zero = gsm + NS * 5 * FRAME_BYTES;
    for (int i = threadIdx.x; i < FRAME_BYTES / 16; i += 32)
        reinterpret_cast<uint4 *>(zero)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const uint32_t base_s = smem_u32(gsm), zero_s = smem_u32(zero);
    int32_t slots[NS][5];
    auto issue = [&](int64_t b, int s) {
        const int32_t *rec = records + idx[b] * REC_INTS;
        int32_t f[REC_INTS];
#pragma unroll
        for (int k = 0; k < REC_INTS; ++k) f[k] = rec[k];
        uint32_t bytes = 0;
#pragma unroll
        for (int fr = 0; fr < 5; ++fr) {
            slots[s][fr] = f[fr];
            if (f[fr] >= 0) bytes += FRAME_BYTES;
        }
        mbar_expect_tx(&bars[s], bytes);
#pragma unroll
        for (int fr = 0; fr < 5; ++fr)
            if (f[fr] >= 0)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        base_s + (uint32_t)((s * 5 + fr) * FRAME_BYTES)),
                    "l"(ring + (size_t)f[fr] * FRAME_BYTES), "r"((uint32_t)FRAME_BYTES), "r"(smem_u32(&bars[s]))
                    : "memory");
        a_out[b] = rec_action(f[5]);
        r_out[b] = rec_reward(f[6], f[7]);
        term_out[b] = (uint8_t)rec_terminal(f[5]);
    };
    auto store = [&](uint8_t *dst, uint32_t src) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
                     "r"((uint32_t)FRAME_BYTES)
                     : "memory");
    };
    const int64_t first = blockIdx.x, stride = gridDim.x;
#pragma unroll
    for (int s = 0; s < NS; ++s)
        if (first + s * stride < B) issue(first + s * stride, s);
    for (int64_t k = 0;; ++k) {
        const int64_t b = first + k * stride;
        if (b >= B) break;
        const int s = (int)(k % NS);
        mbar_wait(&bars[s], (uint32_t)((k / NS) & 1));
#pragma unroll
        for (int fr = 0; fr < 5; ++fr) {
            const uint32_t src = slots[s][fr] >= 0 ? base_s + (uint32_t)((s * 5 + fr) * FRAME_BYTES) : zero_s;
            if (fr < 4) store(s_out + ((size_t)b * 4 + fr) * FRAME_BYTES, src);
            if (fr > 0) store(s2_out + ((size_t)b * 4 + fr - 1) * FRAME_BYTES, src);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // refill the stage written out one iteration ago (its store group has been
        // reading for a whole iteration; the newest group stays in flight)
        if (k >= 1) {
            const int64_t nb = first + (k - 1 + NS) * stride;
            if (nb < B) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                issue(nb, (int)((k - 1) % NS));
            }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ flush
// sampler j's staged steps [k0, k1) -> slots push_count + j * (k1 - k0) + (k - k0)
// (ReplayMemory.flush, replay.py:82-93: ascending owner id, each chronological)
__global__ void k_flush(const int32_t *staging, int W, int steps, int k0, int k1, int32_t *records,
                        int64_t capacity, int64_t push_count) {
    const int len = k1 - k0;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // owner-major index
    if (i >= (int64_t)W * len) return;
    const int64_t j = i / len, k = k0 + (i - j * len);
    int64_t slot = (push_count + i) % capacity;
    const uint4 *src = reinterpret_cast<const uint4 *>(staging + (j * steps + k) * REC_INTS);
    uint4 *dst = reinterpret_cast<uint4 *>(records + slot * REC_INTS);
    dst[0] = src[0];
    dst[1] = src[1];
}

// ------------------------------------------------------------------ frames
__device__ __forceinline__ uint64_t frame_base(uint64_t key, int64_t episode, int t, int action) {
    return splitmix64(splitmix64(splitmix64(key) ^ (uint64_t)episode) ^
                      (((uint64_t)t << 8) | (uint64_t)action));
}

// frame words: word p = splitmix64(base + p) (little-endian bytes = 8 pixels)
__device__ __forceinline__ void write_frame(uint8_t *dst, uint64_t base, int tid, int nthreads) {
    uint64_t *d = reinterpret_cast<uint64_t *>(dst);
    for (int p = tid; p < FRAME_BYTES / 8; p += nthreads) d[p] = splitmix64(base + (uint64_t)p);
}

// prepopulation, sequential part: one thread walks the PREPOP stream exactly like
// replay.py:68-80 with the synthetic frame env (oracle/envs.py)
struct FrameDesc {
    int64_t episode;
    int32_t t, action;
};

__global__ void k_prepop_scalar(uint64_t *pcg, int L, int A, double term_p, int64_t n,
                                int64_t frame_base_seq, int64_t frame_capacity, int32_t *rec,
                                FrameDesc *desc, int64_t *frames_used) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Pcg64 g;
    g.load(pcg);
    int64_t episode = 0, used = 0;
    int t = 0;
    int32_t stack[4];
    auto alloc = [&](int64_t ep, int tt, int a) -> int32_t {
        desc[used] = FrameDesc{ep, tt, a};
        int32_t slot = (int32_t)((frame_base_seq + used) % frame_capacity);
        ++used;
        return slot;
    };
    stack[0] = stack[1] = stack[2] = -1;
    stack[3] = alloc(episode, 0, 255);
    for (int64_t i = 0; i < n; ++i) {
        int a = (int)g.bounded((uint32_t)A);
        double reward = g.random();
        bool term = g.random() < term_p;
        t += 1;
        int32_t fs = alloc(episode, t, a);
        bool trunc = !term && t >= L;
        int32_t *r = rec + i * REC_INTS;
        r[0] = stack[0], r[1] = stack[1], r[2] = stack[2], r[3] = stack[3], r[4] = fs;
        // action | bootstrap terminal (= terminal and not truncated) << 16, f64 reward
        rec_pack(r + 5, a, term, reward);
        if (term || trunc) {
            if (i + 1 < n) {
                episode += 1;
                t = 0;
                stack[0] = stack[1] = stack[2] = -1;
                stack[3] = alloc(episode, 0, 255);
            }
        } else {
            stack[0] = stack[1], stack[1] = stack[2], stack[2] = stack[3], stack[3] = fs;
        }
    }
    g.store(pcg);
    *frames_used = used;
}

__global__ void __launch_bounds__(128) k_gen_frames(const FrameDesc *desc, const int64_t *count,
                                                    uint64_t key, uint8_t *ring,
                                                    int64_t frame_base_seq, int64_t frame_capacity) {
    for (int64_t f = blockIdx.x; f < *count; f += gridDim.x) {
        FrameDesc d = desc[f];
        int64_t slot = (frame_base_seq + f) % frame_capacity;
        write_frame(ring + slot * FRAME_BYTES, frame_base(key, d.episode, d.t, d.action),
                    threadIdx.x, blockDim.x);
    }
}

}  // namespace pq

using namespace pq;

extern "C" {

int pq_sample_indices(uint64_t *pcg_state, uint32_t n, int64_t count, int64_t *idx_out,
                      void *stream) {
    if (n == 0) return set_err("cannot sample from an empty replay memory");
    k_sample_indices<<<1, SAMPLE_THREADS, 0, (cudaStream_t)stream>>>(pcg_state, n, count, idx_out);
    return cuda_err(cudaGetLastError(), "sample_indices");
}

int pq_replay_gather_ldg(const uint8_t *ring, const int32_t *records, const int64_t *idx, int64_t B,
                         uint8_t *s_out, uint8_t *s2_out, int32_t *a_out, double *r_out,
                         uint8_t *term_out, void *stream) {
    if (B <= 0) return 0;
    k_gather<<<(unsigned)B, 256, 0, (cudaStream_t)stream>>>(ring, records, idx, s_out, s2_out,
                                                            a_out, r_out, term_out);
    return cuda_err(cudaGetLastError(), "gather");
}

int pq_replay_gather_tma(const uint8_t *ring, const int32_t *records, const int64_t *idx, int64_t B,
                         uint8_t *s_out, uint8_t *s2_out, int32_t *a_out, double *r_out,
                         uint8_t *term_out, void *stream) {
    if (B <= 0) return 0;
    constexpr int NS = 3;
    constexpr int smem = (NS * 5 + 1) * FRAME_BYTES;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        PQ_CHECK(cudaGetDevice(&dev), "device");
        PQ_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
        PQ_CHECK(cudaFuncSetAttribute(k_gather_tma<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                 "gather smem");
    }
    const int64_t grid = B < 2 * sms ? B : 2 * sms;
    k_gather_tma<NS><<<(unsigned)grid, 32, smem, (cudaStream_t)stream>>>(ring, records, idx, B, s_out, s2_out,
                                                                          a_out, r_out, term_out);
    return cuda_err(cudaGetLastError(), "gather (TMA)");
}

// the product entry point: the 16-byte-load gather (measured 0.97 of HBM peak vs 0.90 for
// the bulk-copy engine: a streaming copy with no reuse gains nothing from the shared-memory
// hop); PQ_GATHER=tma selects the TMA engine
int pq_replay_gather(const uint8_t *ring, const int32_t *records, const int64_t *idx, int64_t B,
                     uint8_t *s_out, uint8_t *s2_out, int32_t *a_out, double *r_out,
                     uint8_t *term_out, void *stream) {
    static int ldg = -1;
    if (ldg < 0) {
        const char *e = getenv("PQ_GATHER");
        ldg = (e && e[0] == 't') ? 0 : 1;
    }
    return (ldg ? pq_replay_gather_ldg : pq_replay_gather_tma)(ring, records, idx, B, s_out, s2_out, a_out,
                                                               r_out, term_out, stream);
}

int pq_replay_flush_range(const int32_t *staging, int W, int steps, int k0, int k1, int32_t *records,
                          int64_t capacity, int64_t push_count, void *stream) {
    if (k0 < 0 || k1 > steps || k0 > k1) return set_err("flush range outside the staged steps");
    int64_t total = (int64_t)W * (k1 - k0);
    if (total <= 0) return 0;
    k_flush<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        staging, W, steps, k0, k1, records, capacity, push_count);
    return cuda_err(cudaGetLastError(), "flush");
}

int pq_replay_flush(const int32_t *staging, int W, int steps, int32_t *records, int64_t capacity,
                    int64_t push_count, void *stream) {
    return pq_replay_flush_range(staging, W, steps, 0, steps, records, capacity, push_count, stream);
}

size_t pq_prepopulate_scratch_bytes(int64_t n) { return (size_t)(2 * n + 2) * sizeof(FrameDesc); }

int pq_prepopulate_walk(uint64_t *pcg_state, int episode_length, int actions, double terminal_p,
                        int64_t n, int64_t frame_base, int64_t frame_capacity, int32_t *rec_out,
                        int64_t *frames_used_out, void *scratch, void *stream) {
    if (n <= 0) return 0;
    k_prepop_scalar<<<1, 32, 0, (cudaStream_t)stream>>>(pcg_state, episode_length, actions, terminal_p, n,
                                                        frame_base, frame_capacity, rec_out,
                                                        static_cast<FrameDesc *>(scratch), frames_used_out);
    return cuda_err(cudaGetLastError(), "prepopulate walk");
}

int pq_prepopulate_frames(uint64_t key, uint8_t *ring, int64_t frame_base, int64_t frame_capacity,
                          const int64_t *frames_used, const void *scratch, void *stream) {
    k_gen_frames<<<4096, 128, 0, (cudaStream_t)stream>>>(static_cast<const FrameDesc *>(scratch), frames_used,
                                                         key, ring, frame_base, frame_capacity);
    return cuda_err(cudaGetLastError(), "prepopulate frames");
}

int pq_prepopulate(uint64_t *pcg_state, uint64_t key, int episode_length, int actions,
                   double terminal_p, int64_t n, uint8_t *ring, int64_t frame_base,
                   int64_t frame_capacity, int32_t *rec_out, int64_t *frames_used_out,
                   void *scratch, void *stream) {
    if (n <= 0) return 0;
    if (int rc = pq_prepopulate_walk(pcg_state, episode_length, actions, terminal_p, n, frame_base,
                                     frame_capacity, rec_out, frames_used_out, scratch, stream))
        return rc;
    return pq_prepopulate_frames(key, ring, frame_base, frame_capacity, frames_used_out, scratch, stream);
}

}  // extern "C"
