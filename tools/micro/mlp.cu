// Issue/complete latency of K independent 16-B loads per lane (32 distinct lines per
// instruction), for ld.global.cg / .ca / default, from one warp or 5 warps per SM.
#include <cstdio>
#include <vector>
#include <random>
typedef unsigned long long u64;
typedef unsigned int u32;
template <int MODE, int K>
__global__ void mlp(const ulonglong2 *buf, u32 mask, int iters, u64 *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = (blockIdx.x * 7919u + warp * 104729u + lane * 15485863u) | 1u;
    long long ti = 0, tc = 0;
    u64 acc = 0;
    for (int it = 0; it < iters; it++) {
        unsigned a[K];
#pragma unroll
        for (int j = 0; j < K; j++) { x = x * 1664525u + 1013904223u; a[j] = (x >> 4) & mask; }
        __syncwarp();
        long long t0 = clock64();
        ulonglong2 v[K];
#pragma unroll
        for (int j = 0; j < K; j++) {
            if (MODE == 0) v[j] = __ldcg(buf + a[j]);
            else if (MODE == 1) v[j] = __ldca(buf + a[j]);
            else v[j] = buf[a[j]];
        }
        long long t1 = clock64();
#pragma unroll
        for (int j = 0; j < K; j++) acc += v[j].x ^ v[j].y;
        acc = __shfl_sync(0xffffffffu, acc, 0);
        long long t2 = clock64();
        ti += t1 - t0; tc += t2 - t0;
        x ^= (unsigned)acc;
    }
    if (lane == 0) { out[(blockIdx.x * 32 + warp) * 2] = ti; out[(blockIdx.x * 32 + warp) * 2 + 1] = tc + (acc == 7 ? 1 : 0); }
}
template <int MODE, int K>
void run(const ulonglong2 *d, u32 mask, int W, int ctas, u64 *o, const char *name) {
    const int iters = 200;
    mlp<MODE, K><<<ctas, 32 * W>>>(d, mask, iters, o);
    mlp<MODE, K><<<ctas, 32 * W>>>(d, mask, iters, o);
    cudaDeviceSynchronize();
    std::vector<u64> r(ctas * 64);
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    double si = 0, sc = 0; int c = 0;
    for (int b = 0; b < ctas; b++) for (int w = 0; w < W; w++) { si += r[(b * 32 + w) * 2]; sc += r[(b * 32 + w) * 2 + 1]; c++; }
    printf("%-8s K=%2d W=%d ctas=%2d footprint=%4u MB: issue %6.0f  complete %6.0f cycles\n", name, K, W, ctas,
           (mask + 1) * 16 >> 20, si / c / iters, sc / c / iters);
}
int main() {
    const size_t n = 1 << 24;   // 256 MB of 16-byte records
    ulonglong2 *d; u64 *o;
    cudaMalloc(&d, n * sizeof(ulonglong2)); cudaMalloc(&o, 148 * 64 * 8);
    cudaMemset(d, 1, n * sizeof(ulonglong2));
    for (u32 mask : {(1u << 18) - 1, (1u << 22) - 1, (1u << 24) - 1}) {   // 4 MB, 64 MB, 256 MB
        run<0, 1>(d, mask, 1, 16, o, "cg"); run<0, 3>(d, mask, 1, 16, o, "cg"); run<0, 16>(d, mask, 1, 16, o, "cg");
        run<0, 3>(d, mask, 5, 16, o, "cg"); run<0, 16>(d, mask, 5, 16, o, "cg");
        run<1, 3>(d, mask, 1, 16, o, "ca"); run<1, 16>(d, mask, 1, 16, o, "ca");
        run<2, 3>(d, mask, 1, 16, o, "default"); run<2, 16>(d, mask, 1, 16, o, "default");
    }
    return 0;
}
