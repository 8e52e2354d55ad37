// l2_store_probe.cu — L2-resident write rate by store form: 16 B st.global per thread (the
// WHT passes' form) against TMA bulk stores (cp.async.bulk.global.shared::cta) of S bytes from
// shared memory. Buffers of 32/64 MiB stay in L2; bytes written per second.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2s l2_store_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void st16(double2* __restrict__ b, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            b[i] = make_double2(r, i);
}

__global__ void st16_v2(double2* __restrict__ b, size_t n, int reps) {  // 2 x 16 B per lane, adjacent
    for (int r = 0; r < reps; ++r)
        for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 2; i < n; i += (size_t)gridDim.x * blockDim.x * 2) {
            b[i] = make_double2(r, i);
            b[i + 1] = make_double2(r, i + 1);
        }
}

// each CTA owns a 32 KiB smem tile and writes it with bulk stores of S bytes over its share
template <unsigned S>
__global__ void bulk(char* __restrict__ b, size_t bytes, int reps) {
    extern __shared__ __align__(128) char sm[];
    constexpr unsigned kTile = 32768;
    for (unsigned i = threadIdx.x; i < kTile / 16; i += blockDim.x)
        reinterpret_cast<double2*>(sm)[i] = make_double2(i, blockIdx.x);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const size_t per_cta = bytes / gridDim.x;
    char* base = b + blockIdx.x * per_cta;
    const unsigned lane = threadIdx.x;
    for (int r = 0; r < reps; ++r) {
        // every thread issues some of the copies (S bytes each), round-robin
        for (size_t off = static_cast<size_t>(lane) * S; off < per_cta; off += static_cast<size_t>(blockDim.x) * S) {
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm + (off % kTile)));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(base + off), "r"(src), "r"(S) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float time_it(F f) {
    cudaEvent_t a, c;
    cudaEventCreate(&a);
    cudaEventCreate(&c);
    f();
    cudaEventRecord(a);
    f();
    cudaEventRecord(c);
    cudaEventSynchronize(c);
    float ms;
    cudaEventElapsedTime(&ms, a, c);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t mib : {32, 64}) {
        const size_t bytes = mib << 20, n = bytes / 16;
        char* b;
        cudaMalloc(&b, bytes);
        cudaMemset(b, 0, bytes);
        const int reps = 50;
        const double tot = double(bytes) * reps;
        float ms = time_it([&] { st16<<<sms * 8, 256>>>(reinterpret_cast<double2*>(b), n, reps); });
        printf("%zu MiB: st.global 16 B/lane      %6.2f TB/s\n", mib, tot / (ms * 1e-3) / 1e12);
        ms = time_it([&] { st16_v2<<<sms * 8, 256>>>(reinterpret_cast<double2*>(b), n, reps); });
        printf("%zu MiB: st.global 2x16 B/lane    %6.2f TB/s\n", mib, tot / (ms * 1e-3) / 1e12);
#define BULK(S, T)                                                                                       \
        cudaFuncSetAttribute(bulk<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);                \
        for (int ctas : {128, 256, 512}) {                                                        \
            ms = time_it([&] { bulk<S><<<ctas, T, 32768>>>(b, bytes, reps); });                            \
            printf("%zu MiB: bulk store %5u B x %3d thr, %4d CTAs %6.2f TB/s\n", mib, S, T, ctas, tot / (ms * 1e-3) / 1e12); \
        }
        BULK(512, 32) BULK(2048, 32) BULK(8192, 32) BULK(512, 128) BULK(2048, 128)
        cudaFree(b);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
