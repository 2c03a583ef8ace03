// Does a kernel launched with programmatic stream serialization honour a preceding
// cudaStreamWaitEvent?  A: slow kernel sets *flag = 1 at its end; B: waits for A's event,
// then launches a PDL kernel that records *flag at its start (and after griddepcontrol.wait).
// Measured on B200 (driver 580): 0/20 early reads in every variant -- the cross-stream joins
// of the fork / join learner schedule (qnet.cu backward_and_update) hold under PDL.
// nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/pdl_event_probe.x scripts/pdl_event_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void slow(volatile int *flag, long long ns) {
    long long t0 = clock64();
    while (clock64() - t0 < ns) {}
    __threadfence();
    *flag = 1;
}
__global__ void tiny(int *x) { if (x) x[1] = 0; }
__global__ void reader(volatile int *flag, int *out) {
    out[0] = *flag;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    out[1] = *flag;
}
int main() {
    int *flag, *out;
    cudaMalloc(&flag, 4); cudaMalloc(&out, 8);
    cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (int pdl = 0; pdl < 2; ++pdl) for (int prev = 0; prev < 2; ++prev) {
        int bad0 = 0, bad1 = 0;
        for (int it = 0; it < 20; ++it) {
            cudaMemset(flag, 0, 4); cudaMemset(out, 0, 8); cudaDeviceSynchronize();
            if (prev) tiny<<<1, 1, 0, b>>>(nullptr);  // a kernel on b before the wait
            slow<<<1, 1, 0, a>>>(flag, 200000000LL / 1000 * 50);  // ~50 us at 2 GHz
            cudaEventRecord(ev, a);
            cudaStreamWaitEvent(b, ev, 0);
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = 1; cfg.blockDim = 1; cfg.stream = b;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = pdl;
            cudaLaunchKernelEx(&cfg, reader, (volatile int *)flag, out);
            cudaDeviceSynchronize();
            int h[2]; cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
            bad0 += h[0] == 0; bad1 += h[1] == 0;
        }
        printf("pdl=%d prev_kernel_on_b=%d: flag unset at start %d/20, after griddepcontrol.wait %d/20\n", pdl, prev, bad0, bad1);
    }
    return 0;
}
