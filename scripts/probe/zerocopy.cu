// zerocopy.cu -- probe: GPU reads of pinned host memory over PCIe (UVA zero-copy):
// sequential coalesced, and one W-byte window per lane at a stride (list heads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int W>
__global__ void k_win(const uint4* __restrict__ h, uint64_t nwin, uint64_t stride16, uint32_t* out)
{
    uint32_t acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwin; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4* p = h + i * stride16;
#pragma unroll
        for (int k = 0; k < W / 16; ++k) { uint4 v = p[k]; acc += v.x ^ v.w; }
    }
    if (acc == 0x12345) *out = acc;
}
__global__ void k_seq(const uint4* __restrict__ h, uint64_t n16, uint32_t* out)
{
    uint32_t acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = h[i]; acc += v.x ^ v.w;
    }
    if (acc == 0x12345) *out = acc;
}
int main() {
    const size_t bytes = 4ull << 30;
    void* h; cudaHostAlloc(&h, bytes, cudaHostAllocMapped); memset(h, 1, bytes);
    uint4* d; cudaHostGetDevicePointer((void**)&d, h, 0);
    uint32_t* o; cudaMalloc(&o, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    for (int g : {sms * 8, sms * 32}) {
        cudaEventRecord(a); k_seq<<<g, 256>>>(d, bytes / 16, o); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("grid %5d sequential: %.1f GB/s\n", g, bytes / ms / 1e6);
        for (int stride : {8, 16, 64}) {            // 16-byte units between windows: 128 B, 256 B, 1 KB
            const uint64_t nwin = bytes / 16 / stride;
            cudaEventRecord(a); k_win<16><<<g, 256>>>(d, nwin, stride, o); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            float w16 = nwin / ms / 1e6;
            cudaEventRecord(a); k_win<32><<<g, 256>>>(d, nwin, stride, o); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            float w32 = nwin / ms / 1e6;
            cudaEventRecord(a); k_win<64><<<g, 256>>>(d, nwin, stride, o); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            float w64 = nwin / ms / 1e6;
            printf("grid %5d stride %4d B: windows/s 16B %.2f G  32B %.2f G  64B %.2f G\n", g, stride * 16, w16, w32, w64);
        }
    }
    return 0;
}
