// L2 bandwidth probe: repeated reads / writes of an L2-resident buffer (bytes per second).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ b, size_t n, int reps, double* sink) {
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(b + i);
            acc += v.x + v.y;
        }
    if (acc == 12345.678) *sink = acc;
}
__global__ void wr(double2* __restrict__ b, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            b[i] = make_double2(r, i);
}
__global__ void rw(double2* __restrict__ b, size_t n, int reps) {
    size_t half = n / 2;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < half; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(b + i);
            b[half + i] = make_double2(v.x + 1, v.y);
        }
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink; cudaMalloc(&sink, 8);
    for (size_t mib : {16, 32, 64}) {
        size_t n = (mib << 20) / 16;
        double2* b; cudaMalloc(&b, n * 16); cudaMemset(b, 0, n * 16);
        cudaEvent_t a, c; cudaEventCreate(&a); cudaEventCreate(&c);
        int reps = 50;
        for (int k = 0; k < 3; ++k) {
            float ms;
            rd<<<sms * 8, 256>>>(b, n, 2, sink);
            cudaEventRecord(a); rd<<<sms * 8, 256>>>(b, n, reps, sink); cudaEventRecord(c); cudaEventSynchronize(c);
            cudaEventElapsedTime(&ms, a, c);
            double rdbw = n * 16.0 * reps / (ms * 1e-3) / 1e12;
            cudaEventRecord(a); wr<<<sms * 8, 256>>>(b, n, reps); cudaEventRecord(c); cudaEventSynchronize(c);
            cudaEventElapsedTime(&ms, a, c);
            double wrbw = n * 16.0 * reps / (ms * 1e-3) / 1e12;
            cudaEventRecord(a); rw<<<sms * 8, 256>>>(b, n, reps); cudaEventRecord(c); cudaEventSynchronize(c);
            cudaEventElapsedTime(&ms, a, c);
            double rwbw = n * 16.0 * reps / (ms * 1e-3) / 1e12;
            printf("%zu MiB: L2 read %.2f TB/s  write %.2f TB/s  read+write %.2f TB/s (bytes moved)\n", mib, rdbw, wrbw, rwbw);
        }
        cudaFree(b);
    }
    return 0;
}
