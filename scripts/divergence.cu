// divergence.cu -- does a lone lane run slowly while its warp siblings wait at __syncthreads?
#include <cstdio>
#include <cstdint>
__global__ void k(int mode, int iters, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = threadIdx.x * 7;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    if (warp == 1) {
        if (mode == 0) {            // lane 0 alone, siblings fall through to __syncthreads
            if (lane == 0) {
                unsigned long long t0 = clock64();
                for (int i = 0; i < iters; i++) acc += tab[i & 63] + i;
                out[0] = clock64() - t0;
            }
        } else if (mode == 1) {     // whole warp runs the loop
            unsigned long long t0 = clock64();
            for (int i = 0; i < iters; i++) acc += tab[i & 63] + i;
            if (lane == 0) out[1] = clock64() - t0;
        } else {                    // lane 0 alone, siblings park at __syncwarp-free exit then bar
            if (lane == 0) {
                unsigned long long t0 = clock64();
                for (int i = 0; i < iters; i++) acc += tab[i & 63] + i;
                out[2] = clock64() - t0;
            }
            __syncwarp();
        }
    }
    sink[threadIdx.x] = acc;
    __syncthreads();
}
int main() {
    unsigned long long* d; uint32_t* s;
    cudaMalloc(&d, 64); cudaMalloc(&s, 4096);
    for (int m = 0; m < 3; m++) k<<<1, 256>>>(m, 10000, d, s);
    cudaDeviceSynchronize();
    unsigned long long h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("cycles/iter: lone-lane-siblings-at-bar %.1f  converged %.1f  lone-lane-then-syncwarp %.1f\n",
           h[0] / 10000.0, h[1] / 10000.0, h[2] / 10000.0);
}
