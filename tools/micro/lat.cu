// Latency microbenchmark: dependent chains of 16-byte loads over a random
// permutation, L1-cached (.ca) vs L2 (.cg), with W active warps per CTA.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
typedef unsigned long long u64;
__global__ void chase(const ulonglong2 *buf, int steps, int mode, u64 *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u64 idx = (blockIdx.x * 977 + warp * 131) % 1024;
    long long t0 = clock64();
    for (int i = 0; i < steps; i++) {
        ulonglong2 v;
        if (mode == 0) v = __ldca(buf + idx + lane * 0);   // one line per warp step
        else if (mode == 1) v = __ldcg(buf + idx);
        else v = __ldca(buf + ((idx + lane * 4099) & ((1 << 20) - 1)));   // 32 distinct lines
        idx = __shfl_sync(0xffffffffu, v.x, 0);
    }
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 32 + warp] = (u64)(t1 - t0) + (idx == 12345678 ? 1 : 0);
}
int main() {
    const int n = 1 << 20;   // 16 MB of 16-byte records
    std::vector<unsigned> perm(n);
    for (int i = 0; i < n; i++) perm[i] = i;
    std::mt19937 g(1);
    std::shuffle(perm.begin(), perm.end(), g);
    std::vector<ulonglong2> h(n);
    for (int i = 0; i < n; i++) { h[perm[i]].x = perm[(i + 1) % n]; h[perm[i]].y = 0; }
    ulonglong2 *d; u64 *o;
    cudaMalloc(&d, n * sizeof(ulonglong2)); cudaMalloc(&o, 148 * 32 * 8);
    cudaMemcpy(d, h.data(), n * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    const int steps = 2000;
    for (int mode = 0; mode < 3; mode++)
        for (int W : {1, 5, 9}) for (int ctas : {1, 16}) {
            chase<<<ctas, 32 * W>>>(d, steps, mode, o);
            chase<<<ctas, 32 * W>>>(d, steps, mode, o);
            cudaDeviceSynchronize();
            std::vector<u64> r(ctas * 32);
            cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
            double s = 0; int c = 0;
            for (int b = 0; b < ctas; b++) for (int w = 0; w < W; w++) { s += r[b * 32 + w]; c++; }
            printf("mode %d (%s) W=%d ctas=%d: %.0f cycles per dependent load\n", mode,
                   mode == 0 ? "ca, 1 line" : mode == 1 ? "cg, 1 line" : "ca, 32 lines", W, ctas, s / c / steps);
        }
    return 0;
}
