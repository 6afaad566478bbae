// Probe (profiling aid, not product): (1) does this host expose NVLS multicast
// objects (cuMulticastCreate / cuMulticastBindMem) and do multimem.st /
// multimem.ld_reduce / multimem.red execute through them; (2) the streaming
// HBM read ceiling with 16-byte non-coherent loads and with TMA bulk loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/nvls_probe scripts/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_ = nullptr; cuGetErrorString(r_, &s_); \
  printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?"); return 1; } } while (0)
#define CR(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void mc_store(float* mc, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float a = i, b = i + 1, c = i + 2, d = i + 3;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}
__global__ void mc_red(float* mc, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float a = 1, b = 1, c = 1, d = 1;
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}
__global__ void mc_ldred(const float* mc, float* out, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + i) : "memory");
    out[i] = a; out[i + 1] = b; out[i + 2] = c; out[i + 3] = d;
  }
}
__global__ void mc_ldred_bf16(const unsigned* mc, unsigned* out, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    unsigned a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc + i) : "memory");
    out[i] = a; out[i + 1] = b; out[i + 2] = c; out[i + 3] = d;
  }
}

// streaming read: 16-byte non-coherent loads, 4 in flight per thread, xor-sum sink
__global__ void __launch_bounds__(512) read_nc(const uint4* __restrict__ p, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { uint4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) *sink = acc;
}

// streaming read through TMA bulk copies into a smem ring (one elected thread issues)
__global__ void __launch_bounds__(32) read_bulk(const char* __restrict__ p, size_t bytes, size_t chunk, int stages, unsigned* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[16];
  if (threadIdx.x != 0) return;
  unsigned nch = (unsigned)(bytes / chunk);
  for (int s = 0; s < stages; ++s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  unsigned it = 0;
  unsigned phase[16] = {0};
  for (unsigned c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    int s = it % stages;
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    if (it >= (unsigned)stages) {
      asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(a), "r"(phase[s]));
      phase[s] ^= 1;
    }
    unsigned dst = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * chunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"((unsigned)chunk));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(p + (size_t)c * chunk), "r"((unsigned)chunk), "r"(a) : "memory");
  }
  for (int s = 0; s < stages && (unsigned)s < it; ++s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(a), "r"(phase[s]));
  }
  if (smem[0] == 123 && smem[1] == 45) *sink = 1;
}

int main() {
  CR(cudaSetDevice(0));
  CR(cudaFree(0));
  int ndev = 0;
  CR(cudaGetDeviceCount(&ndev));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc = 0, fab = 0, vmm = 0, sms = 0;
  CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  printf("devices=%d multicast_supported=%d fabric_handles=%d vmm=%d sms=%d\n", ndev, mc, fab, vmm, sms);

  // ---- HBM streaming read ceiling ----
  {
    size_t bytes = 470ull << 20;
    char* buf;
    unsigned* sink;
    CR(cudaMalloc(&buf, bytes));
    CR(cudaMalloc(&sink, 4));
    CR(cudaMemset(buf, 1, bytes));
    char* flush;
    size_t fb = 512ull << 20;
    CR(cudaMalloc(&flush, fb));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn) {
      float best = 1e30f;
      for (int r = 0; r < 12; ++r) {
        cudaMemsetAsync(flush, r, fb);       // evict the buffer from L2
        cudaMemsetAsync(sink, 0, 4);          // (small write, then a read sweep drains dirty lines)
        cudaEventRecord(e0);
        fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2 && ms < best) best = ms;
      }
      return best;
    };
    for (int cpsm : {2}) {
      for (int thr : {256, 512}) {
        int grid = sms * cpsm * (512 / thr);
        float ms = timeit([&] { read_nc<<<grid, thr>>>((const uint4*)buf, bytes / 16, sink); });
        printf("read_nc grid=%d thr=%d: %.1f us  %.0f GB/s\n", grid, thr, ms * 1e3, bytes / ms / 1e6);
      }
    }
    for (size_t chunk : {32768ull}) {
      for (int stages : {4, 6}) {
        size_t sm = chunk * stages;
        if (sm > 200 * 1024) continue;
        cudaFuncSetAttribute(read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int cpsm : {1, 2}) {
          if (sm * cpsm > 220 * 1024) continue;
          float ms = timeit([&] { read_bulk<<<sms * cpsm, 32, sm>>>(buf, bytes, chunk, stages, sink); });
          printf("read_bulk chunk=%zu stages=%d ctas=%d: %.1f us  %.0f GB/s\n", chunk, stages, sms * cpsm, ms * 1e3, bytes / ms / 1e6);
        }
      }
    }
    CR(cudaGetLastError());
    cudaFree(buf);
    cudaFree(flush);
  }

  if (!mc) {
    printf("NVLS: multicast not supported on this device/host\n");
    return 0;
  }
  // ---- NVLS multicast object over one device ----
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.flags = 0;
  size_t gran = 0, rgran = 0;
  mp.size = 2 << 20;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&rgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t size = ((4u << 20) + rgran - 1) / rgran * rgran;
  mp.size = size;
  printf("mc granularity min=%zu rec=%zu size=%zu\n", gran, rgran, size);
  CUmemGenericAllocationHandle mch;
  {
    CUresult r = CUDA_ERROR_INVALID_VALUE;
    const CUmemAllocationHandleType hts[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_NONE};
    for (unsigned nd : {1u, 2u}) {
      for (auto ht : hts) {
        mp.numDevices = nd;
        mp.handleTypes = ht;
        r = cuMulticastCreate(&mch, &mp);
        const char* s = nullptr;
        cuGetErrorString(r, &s);
        printf("cuMulticastCreate numDevices=%u handleTypes=%d -> %d %s\n", nd, (int)ht, (int)r, s ? s : "?");
        if (r == CUDA_SUCCESS) break;
      }
      if (r == CUDA_SUCCESS) break;
    }
    if (r != CUDA_SUCCESS) return 1;
    if (mp.numDevices != 1) { printf("NVLS: a multicast object needs >1 device here; cannot bind one GPU\n"); }
  }
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  CUmemGenericAllocationHandle mem;
  CK(cuMemCreate(&mem, size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, mem, 0, size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, size, rgran, 0, 0));
  CK(cuMemMap(uc, size, 0, mem, 0));
  CK(cuMemAddressReserve(&mcp, size, rgran, 0, 0));
  CK(cuMemMap(mcp, size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, size, &ad, 1));
  CK(cuMemSetAccess(mcp, size, &ad, 1));
  int n = 1 << 20;
  float* out;
  CR(cudaMalloc(&out, n * 4));
  mc_store<<<n / 4 / 256, 256>>>((float*)mcp, n);
  CR(cudaDeviceSynchronize());
  std::vector<float> h(n);
  CR(cudaMemcpy(h.data(), (void*)uc, n * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != (float)i;
  printf("multimem.st: %s (bad=%d)\n", bad ? "WRONG" : "ok", bad);
  mc_red<<<n / 4 / 256, 256>>>((float*)mcp, n);
  CR(cudaDeviceSynchronize());
  CR(cudaMemcpy(h.data(), (void*)uc, n * 4, cudaMemcpyDeviceToHost));
  bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != (float)i + 1;
  printf("multimem.red.add: %s (bad=%d)\n", bad ? "WRONG" : "ok", bad);
  mc_ldred<<<n / 4 / 256, 256>>>((const float*)mcp, out, n);
  CR(cudaDeviceSynchronize());
  CR(cudaMemcpy(h.data(), out, n * 4, cudaMemcpyDeviceToHost));
  bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != (float)i + 1;
  printf("multimem.ld_reduce.add: %s (bad=%d)\n", bad ? "WRONG" : "ok", bad);
  mc_ldred_bf16<<<n / 4 / 256, 256>>>((const unsigned*)mcp, (unsigned*)out, n);
  CR(cudaDeviceSynchronize());
  // bandwidth of multimem.st / ld_reduce over one device (switch round trip)
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) mc_store<<<n / 4 / 256, 256>>>((float*)mcp, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("multimem.st 4 MiB x10: %.1f us/iter %.0f GB/s\n", ms * 100, n * 4.0 * 10 / ms / 1e6);
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) mc_ldred<<<n / 4 / 256, 256>>>((const float*)mcp, out, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("multimem.ld_reduce 4 MiB x10: %.1f us/iter %.0f GB/s\n", ms * 100, n * 4.0 * 10 / ms / 1e6);
    }
  }
  CR(cudaGetLastError());
  printf("NVLS probe done\n");
  return 0;
}
