// Latency micro-benchmarks on one warp / one CTA (clock64): dependent DFMA, DMUL, double reciprocal (1.0/x),
// dependent DMMA m8n8k4, __shfl_sync of a double, bar.sync over 256 threads, LDS.128 round trip.
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, double seed)
{
    __shared__ double2 sh[512];
    const int N = 1024;
    double x = seed + threadIdx.x, y = 1.0000001, c0 = 0, c1 = 0;
    long long t0, t1;
    sh[threadIdx.x] = make_double2(x, 0);
    __syncthreads();
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < N; i++) x = fma(x, y, 1e-9);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
    // reciprocal chain
    t0 = clock64();
    for (int i = 0; i < N; i++) x = 1.0 / (x + 1e-3);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / N;
    // DMMA chain (same accumulator)
    t0 = clock64();
    for (int i = 0; i < N; i++) dmma(c0, c1, x, y);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0) / N;
    // shfl chain
    t0 = clock64();
    for (int i = 0; i < N; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) / N;
    // bar.sync 256
    t0 = clock64();
    for (int i = 0; i < N; i++) asm volatile("bar.sync 1, 256;" ::: "memory");
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0) / N;
    // dependent LDS.128
    int idx = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < N; i++) {
        double2 v = sh[idx];
        idx = ((int)v.y + idx + 1) & 255;
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0) / N;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < N; i++) x = x * y;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0) / N;
    out[threadIdx.x] = x + c0 + c1 + idx;
}
int main()
{
    double* o;
    long long* c;
    cudaMalloc(&o, 4096 * 8);
    cudaMallocManaged(&c, 16 * 8);
    k<<<1, 256>>>(o, c, 1.0);
    cudaDeviceSynchronize();
    k<<<1, 256>>>(o, c, 1.0);
    cudaDeviceSynchronize();
    printf("DFMA %lld  RCP(1/x incl add) %lld  DMMA %lld  SHFL %lld  BAR256 %lld  LDS128 %lld  DMUL %lld  (cycles, dependent)\n",
           c[0], c[1], c[2], c[3], c[4], c[5], c[6]);
    return 0;
}
