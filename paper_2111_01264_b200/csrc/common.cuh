// Shared device helpers for the sm_100a fast-DQN hot path: PTX wrappers for
// mbarrier / tcgen05 (TMEM alloc, UMMA issue, commit, TMEM load), UMMA smem
// descriptors, bf16 packing and the numpy-compatible PCG64 generator.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#define PQ_DEV __device__ __forceinline__

namespace pq {

// Kernel launch with the programmatic-stream-serialization attribute (PDL) unless
// PQ_PDL=0 is set in the environment.
inline bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("PQ_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on != 0;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- smem / mbarrier
PQ_DEV uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

PQ_DEV void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

PQ_DEV void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

PQ_DEV bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

PQ_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

PQ_DEV void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// barrier among `count` threads (multiple of 32) on hardware barrier `id` (1..15)
PQ_DEV void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// generic-proxy smem writes -> visible to the async proxy (UMMA operand reads)
PQ_DEV void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM
template <uint32_t NCOLS>
PQ_DEV void tmem_alloc(uint32_t *dst_smem) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t NCOLS>
PQ_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
                 : "memory");
}

PQ_DEV void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
PQ_DEV void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate (kind::f16)
PQ_DEV void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// arrive on an mbarrier once every previously issued UMMA of this thread completes
PQ_DEV void umma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// TMEM -> registers: 32 lanes x 32 consecutive 32-bit columns (one per register)
PQ_DEV void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

PQ_DEV void tmem_ld16(uint32_t taddr, float (&v)[32]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
#pragma unroll
    for (int i = 16; i < 32; ++i) v[i] = 0.f;
}

// ---------------------------------------------------------------- UMMA descriptors
// 128B-swizzled canonical layouts (bf16):
//  K-major : rows of 64 K-elements (128 B), 8-row atoms of 1024 B at SBO = 1024.
//  MN-major: rows of 64 MN-elements (128 B) per K index, 8-K-row atoms of 1024 B at
//            SBO = 1024 (K direction), MN atoms at LBO = 64 * 128 B = 8192 (BK = 64).
PQ_DEV uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor: bf16 x bf16 -> f32, M = 128, N, majors
__host__ __device__ constexpr uint32_t idesc_bf16(int N, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// byte offset of the 16-byte chunk (row, chunk) inside a K-major SW128 tile
PQ_DEV uint32_t kmaj_off(int row, int c8) {
    return (uint32_t)(row * 128 + ((c8 ^ (row & 7)) << 4));
}
// byte offset of chunk (k, m8) inside an MN-major SW128 tile with BK = 64
PQ_DEV uint32_t mnmaj_off(int k, int m8) {
    return (uint32_t)((m8 >> 3) * 8192 + (k >> 3) * 1024 + (k & 7) * 128 +
                      (((m8 & 7) ^ (k & 7)) << 4));
}

// ---------------------------------------------------------------- bf16 helpers
PQ_DEV uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
PQ_DEV float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
PQ_DEV float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// 8 unsigned bytes -> 8 bf16 (exact: integers <= 255 are representable)
PQ_DEV uint4 u8x8_to_bf16(uint32_t lo, uint32_t hi) {
    uint4 r;
    r.x = pack_bf16((float)(lo & 0xFF), (float)((lo >> 8) & 0xFF));
    r.y = pack_bf16((float)((lo >> 16) & 0xFF), (float)(lo >> 24));
    r.z = pack_bf16((float)(hi & 0xFF), (float)((hi >> 8) & 0xFF));
    r.w = pack_bf16((float)((hi >> 16) & 0xFF), (float)(hi >> 24));
    return r;
}

// ---------------------------------------------------------------- PCG64 (numpy)
// state layout (u64[6]): state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger
struct U128 {
    uint64_t hi, lo;
};
PQ_DEV U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}
PQ_DEV U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}
__device__ constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ULL;
__device__ constexpr uint64_t PCG_MULT_LO = 0x4385DF649FCCF645ULL;

PQ_DEV uint64_t pcg_output(U128 s) {
    uint64_t x = s.hi ^ s.lo;
    unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct Pcg64 {
    U128 state, inc;
    uint32_t has32, buf;

    PQ_DEV void load(const uint64_t *s) {
        state = {s[0], s[1]};
        inc = {s[2], s[3]};
        has32 = (uint32_t)s[4];
        buf = (uint32_t)s[5];
    }
    PQ_DEV void store(uint64_t *s) const {
        s[0] = state.hi;
        s[1] = state.lo;
        s[2] = inc.hi;
        s[3] = inc.lo;
        s[4] = has32;
        s[5] = buf;
    }
    PQ_DEV uint64_t next64() {
        state = add128(mul128(state, U128{PCG_MULT_HI, PCG_MULT_LO}), inc);
        return pcg_output(state);
    }
    PQ_DEV uint32_t next32() {
        if (has32) {
            has32 = 0;
            return buf;
        }
        uint64_t v = next64();
        has32 = 1;
        buf = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // Generator.random()
    PQ_DEV double random() {
        return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
    }
    // Generator.integers(0, n) for 1 <= n < 2^32 (buffered Lemire, rng = n - 1)
    PQ_DEV uint32_t bounded(uint32_t n) {
        if (n <= 1) return 0;
        uint64_t m = (uint64_t)next32() * n;
        uint32_t left = (uint32_t)m;
        if (left < n) {
            uint32_t threshold = (0u - n) % n;  // (2^32 - n) mod n
            while (left < threshold) {
                m = (uint64_t)next32() * n;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

// LCG jump-ahead by delta steps (pcg_advance_lcg_128)
PQ_DEV U128 pcg_advance(U128 state, U128 inc, uint64_t delta) {
    U128 acc_mult{0, 1}, acc_plus{0, 0}, cur_mult{PCG_MULT_HI, PCG_MULT_LO}, cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult = mul128(acc_mult, cur_mult);
            acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
        }
        cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
        cur_mult = mul128(cur_mult, cur_mult);
        delta >>= 1;
    }
    return add128(mul128(acc_mult, state), acc_plus);
}

// ---------------------------------------------------------------- TMA (cp.async.bulk.tensor)
// Tiled tensor loads into shared memory, completion counted in bytes on an mbarrier.
// `map` is the generic address of a CUtensorMap in parameter / constant / global memory.
PQ_DEV void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
PQ_DEV void tma_load_2d(uint32_t dst, const void *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
PQ_DEV void tma_load_3d(uint32_t dst, const void *map, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
PQ_DEV void tma_load_4d(uint32_t dst, const void *map, uint64_t *bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// im2col load of an NHWC tensor map (cuTensorMapEncodeIm2col): pixelsPerColumn pixels
// from base pixel (n, h, w) walked W -> H -> N through the map's bounding box, each
// contributing channelsPerPixel channels from c, at filter-tap offset (ow, oh).
PQ_DEV void tma_im2col_4d(uint32_t dst, const void *map, uint64_t *bar, int c, int w, int h, int n, uint16_t ow,
                          uint16_t oh) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
        "l"(map), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
        : "memory");
}

// 4 rows (row0..row3, any order, negative / past-the-end = zero-filled) x one box width of
// a 2D tensor map whose box is {width, 1}: Blackwell tile::gather4.  The rows land at
// consecutive box-row positions of dst (swizzled like a 4-row tile box).
PQ_DEV void tma_gather4(uint32_t dst, const void *map, uint64_t *bar, int col, int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(map), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// ---------------------------------------------------------------- programmatic dependent launch
// wait: block until the predecessor grid in the stream has completed (no-op when the
// kernel was launched without the PDL attribute); launch: let the dependent grid start
// its prologue now.  Every kernel triggers right after its own wait, so a dependent
// that starts early may read anything produced two or more kernels back.
PQ_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
PQ_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- timeline probes
// Compiled in only for profiling builds (make probes: -DPQ_PROBES=1 into _lib/probes/);
// the shipped library carries none of their loads or branches.
#ifndef PQ_PROBES
#define PQ_PROBES 0
#endif
constexpr bool kProbes = PQ_PROBES != 0;
// Runtime-gated phase timestamps (%globaltimer, ns) of CTA 0 of each launch plus the
// last CTA's end, for latency analysis (pq_timeline_*).  Off by default.
struct Timeline {
    int on;
    int n;
    unsigned long long t[256][12];
    char tag[256];
    unsigned int ctas[64];  // finished CTAs per (tag, grid) key of the running launches
};
static __device__ Timeline g_tl;  // one copy per translation unit (GEMMs live in qnet.cu)

PQ_DEV unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
PQ_DEV bool tl_cta0() { return blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0; }

// Per-CTA trace (pq_cta_trace): every CTA's thread 0 records its start, dependency
// release, accumulator-ready and end times plus SM id, linear CTA index, kernel tag and
// grid size.  Runtime-gated, off by default.
struct CtaTrace {
    int on;
    unsigned n;
    unsigned long long r[8192][6];
};
static __device__ CtaTrace g_ct;
static __shared__ unsigned long long s_ct[3];
static __shared__ int s_ct_on;  // thread 0's copy of g_ct.on (read once per CTA)
PQ_DEV void ct_begin() {
    if (!kProbes) return;
    if (threadIdx.x == 0) {
        s_ct_on = g_ct.on;
        if (s_ct_on) s_ct[0] = gtime(), s_ct[1] = 0ull, s_ct[2] = 0ull;
    }
}
PQ_DEV void ct_mark(int i) {
    if (kProbes && threadIdx.x == 0 && s_ct_on) s_ct[i] = gtime();
}
PQ_DEV void ct_end(char tag, int part = 0) {
    if (!kProbes || threadIdx.x != 0 || !s_ct_on) return;
    const unsigned long long t = gtime();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned slot = atomicAdd(&g_ct.n, 1u);
    if (slot >= 8192) return;
    const unsigned lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    g_ct.r[slot][0] = s_ct[0], g_ct.r[slot][1] = s_ct[1], g_ct.r[slot][2] = s_ct[2], g_ct.r[slot][3] = t;
    g_ct.r[slot][4] = ((unsigned long long)smid << 32) | lin;
    g_ct.r[slot][5] = ((unsigned long long)(unsigned char)tag << 48) | ((unsigned long long)part << 40) | total;
}
// slots 8..11 of a record: grid dims and a kernel tag (identify the launch)
PQ_DEV void tl_ident(int slot, char tag) {
    g_tl.t[slot][8] = gridDim.x, g_tl.t[slot][9] = gridDim.y, g_tl.t[slot][10] = gridDim.z;
    g_tl.t[slot][11] = (unsigned long long)tag;
    g_tl.tag[slot] = tag;
}
// every CTA's thread 0 at its very end: the last CTA of a launch appends an 'E' record
// (end time, grid dims, tag in slot 7) -- matched to the launch by grid and order
PQ_DEV void tl_cta_end(char tag) {
    if (!kProbes || !g_tl.on || threadIdx.x != 0) return;
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    const unsigned key = (gridDim.x * 131u + gridDim.y * 7u + gridDim.z * 3u + (unsigned)tag) & 63u;
    __threadfence();
    if (atomicAdd(&g_tl.ctas[key], 1u) + 1 == total) {
        const unsigned long long t = gtime();
        g_tl.ctas[key] = 0;
        const int slot = atomicAdd(&g_tl.n, 1);
        if (slot < 256) {
            for (int k = 0; k < 8; ++k) g_tl.t[slot][k] = k == 0 ? t : k == 7 ? (unsigned long long)tag : 0ull;
            tl_ident(slot, 'E');
        }
    }
}
// start / predecessor-done / end stamps of CTA 0 of a non-GEMM kernel (same slot layout)
struct TlProbe {
    bool on;
    unsigned long long t0, t1;
    PQ_DEV TlProbe() : on(kProbes && g_tl.on && tl_cta0() && threadIdx.x == 0), t0(on ? gtime() : 0ull), t1(0ull) {}
    PQ_DEV void waited() {
        if (on) t1 = gtime();
    }
    PQ_DEV void done(char tag) {
        tl_cta_end(tag);
        if (!on) return;
        const unsigned long long t2 = gtime();
        const int slot = atomicAdd(&g_tl.n, 1);
        if (slot < 256) {
            for (int k = 0; k < 8; ++k) g_tl.t[slot][k] = k == 0 ? t0 : k == 1 ? t1 : k == 2 ? t2 : 0ull;
            tl_ident(slot, tag);
        }
    }
};

// ---------------------------------------------------------------- misc
PQ_DEV uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace pq
