// SM-partitioned streams (green contexts): a stream whose kernels run on a fixed subset of
// the GPU's SMs.  The executor can put the acting stream on such a partition so the
// lockstep acting blocks never take the SMs the learner's full-width grids are waiting
// for (PQ_ACT_SMS).  Driver entry points come through cudaGetDriverEntryPoint, so the
// library does not link libcuda directly.
#include <cuda.h>
#include <cuda_runtime.h>

namespace pq {
int set_err(const char *msg);
}

namespace {

template <class F>
int entry(const char *name, F *fn) {
    cudaDriverEntryPointQueryResult q{};
    void *p = nullptr;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p ||
        q != cudaDriverEntryPointSuccess)
        return 1;
    *fn = reinterpret_cast<F>(p);
    return 0;
}

}  // namespace

extern "C" int pq_sm_partition_stream(int sm_count, void **stream_out, int *sm_granted) {
    using DevGet = CUresult (*)(CUdevice *, int);
    using GetRes = CUresult (*)(CUdevice, CUdevResource *, CUdevResourceType);
    using Split = CUresult (*)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *, unsigned,
                               unsigned);
    using Desc = CUresult (*)(CUdevResourceDesc *, CUdevResource *, unsigned);
    using Green = CUresult (*)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned);
    using GStream = CUresult (*)(CUstream *, CUgreenCtx, unsigned, int);
    DevGet dev_get;
    GetRes get_res;
    Split split;
    Desc desc_fn;
    Green green;
    GStream gstream;
    if (entry("cuDeviceGet", &dev_get) || entry("cuDeviceGetDevResource", &get_res) ||
        entry("cuDevSmResourceSplitByCount", &split) || entry("cuDevResourceGenerateDesc", &desc_fn) ||
        entry("cuGreenCtxCreate", &green) || entry("cuGreenCtxStreamCreate", &gstream))
        return pq::set_err("green-context driver entry points unavailable");
    if (sm_count < 1 || !stream_out) return pq::set_err("sm_count must be >= 1");
    int ord = 0;
    if (cudaGetDevice(&ord) != cudaSuccess) return pq::set_err("no current device");
    cudaFree(nullptr);  // the primary context exists before the partition is carved
    CUdevice dev;
    CUdevResource all{}, part{}, rest{};
    unsigned n = 1;
    CUdevResourceDesc desc;
    CUgreenCtx g;
    CUstream s;
    if (dev_get(&dev, ord) != CUDA_SUCCESS || get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
        return pq::set_err("cuDeviceGetDevResource failed");
    if (split(&part, &n, &all, &rest, 0, (unsigned)sm_count) != CUDA_SUCCESS || n != 1)
        return pq::set_err("cuDevSmResourceSplitByCount failed");
    if (desc_fn(&desc, &part, 1) != CUDA_SUCCESS) return pq::set_err("cuDevResourceGenerateDesc failed");
    if (green(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return pq::set_err("cuGreenCtxCreate failed");
    if (gstream(&s, g, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return pq::set_err("cuGreenCtxStreamCreate failed");
    *stream_out = (void *)s;
    if (sm_granted) *sm_granted = (int)part.sm.smCount;
    return 0;
}
