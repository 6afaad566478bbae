// Probe: do same-device D2D copies make progress while a persistent kernel
// occupies every SM (~200 KB smem/CTA)? Each variant: spin kernel waits for a
// flag that a copy stream writes (cuStreamWriteValue32) after the copy.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <chrono>

__global__ void spin(volatile unsigned* flag, unsigned target, unsigned long long timeout_ns, int* result) {
    extern __shared__ char sm[];
    sm[threadIdx.x] = 0;
    unsigned long long t0; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    while (*flag < target) {
        unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) { if (threadIdx.x == 0) atomicAdd(result, 1); return; }
        __nanosleep(1000);
    }
}

int main() {
    PFN_cuStreamWriteValue32_v11070 wv; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&wv, cudaEnableDefault, &q);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t bytes = 8 << 20;
    char *a, *b; cudaMalloc(&a, bytes * 2); cudaMalloc(&b, bytes * 2);
    int dev1 = 0; 
    unsigned* flag; cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
    int* res; cudaMalloc(&res, 4);
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t ks, cs; cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    const char* names[] = {"memcpyAsync 1D D2D", "memcpy2DAsync D2D", "memcpyPeerAsync same dev", "memcpyAsync 1D D2D 64MB"};
    for (int v = 0; v < 4; ++v) {
        cudaMemset(res, 0, 4);
        cudaDeviceSynchronize();
        spin<<<sms, 256, 200 * 1024, ks>>>(flag, v + 1, 3000000000ull, res);
        auto t0 = std::chrono::steady_clock::now();
        cudaError_t e;
        if (v == 0) e = cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice, cs);
        else if (v == 1) e = cudaMemcpy2DAsync(b, 16384, a, 16384, 16384, bytes / 16384, cudaMemcpyDeviceToDevice, cs);
        else if (v == 2) e = cudaMemcpyPeerAsync(b, dev1, a, dev1, bytes, cs);
        else e = cudaMemcpyAsync(b, a, bytes * 2, cudaMemcpyDeviceToDevice, cs);
        wv((CUstream)cs, (CUdeviceptr)flag, v + 1, 0);
        cudaStreamSynchronize(cs);
        double copy_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        cudaStreamSynchronize(ks);
        int r = -1; cudaMemcpy(&r, res, 4, cudaMemcpyDeviceToHost);
        printf("%-28s launch=%s copy+flag %.3f ms, spin CTAs timed out: %d/%d\n", names[v], cudaGetErrorString(e), copy_ms, r, sms);
    }
    // copy bandwidth with idle SMs, CE-style 1D vs 2D
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int v = 0; v < 2; ++v) {
        cudaEventRecord(e0, cs);
        for (int i = 0; i < 10; ++i)
            if (v == 0) cudaMemcpyAsync(b, a, bytes * 2, cudaMemcpyDeviceToDevice, cs);
            else cudaMemcpy2DAsync(b, 16384, a, 16384, 16384, bytes * 2 / 16384, cudaMemcpyDeviceToDevice, cs);
        cudaEventRecord(e1, cs); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%s 16MB x10: %.1f GB/s (read+write)\n", v ? "2D" : "1D", 2.0 * 10 * bytes * 2 / (ms * 1e-3) / 1e9);
    }
    return 0;
}
