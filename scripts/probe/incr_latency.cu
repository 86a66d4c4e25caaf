// incr_latency.cu -- per-call cost of cc_incr_batch for small batches (Table 5's
// latency regime), measured from C so that no Python overhead is
// included: B calls back to back on one stream with device-resident batches,
// CUDA events around the loop (device time per call) and steady_clock around
// the issue loop (host time per call).  Build: make probes.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/cc.h"

static uint64_t sm64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

int main(int argc, char** argv)
{
    const uint32_t n = 1u << 20;
    const int calls = argc > 1 ? atoi(argv[1]) : 4000;
    const int sizes[] = {1, 10, 100, 1000, 10000};
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int bs : sizes) {
        std::vector<uint32_t> h(2 * (size_t)bs * calls);
        for (size_t i = 0; i < h.size(); ++i) h[i] = (uint32_t)((sm64(i + 77 * bs) & 0xFFFFFFFFull) * n >> 32);
        uint32_t* d = nullptr;
        cudaMalloc(&d, 4 * h.size());
        cudaMemcpy(d, h.data(), 4 * h.size(), cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 2; ++rep) {
            cc_incr* hd = nullptr;
            cc_incr_create(n, nullptr, s, &hd);
            cudaStreamSynchronize(s);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            const auto t0 = std::chrono::steady_clock::now();
            for (int c = 0; c < calls; ++c) {
                const cc_status rc = cc_incr_batch(hd, d + 2 * (size_t)bs * c, bs, nullptr, 0, nullptr, s);
                if (rc) { printf("rc=%d %s\n", rc, cc_last_error()); return 1; }
            }
            const auto t1 = std::chrono::steady_clock::now();
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / calls;
            if (rep)
                printf("{\"batch\": %d, \"calls\": %d, \"us_per_call_device\": %.3f, \"us_per_call_host_issue\": %.3f, "
                       "\"inserts_per_s\": %.4g}\n", bs, calls, 1e3 * ms / calls, host_us, bs * calls / (ms * 1e-3));
            cc_incr_destroy(hd);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        cudaFree(d);
    }
    return 0;
}
