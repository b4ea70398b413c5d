// LDS.128 bank-conflict model probe: lane l reads the 16-byte chunk (l & 3) of
// a 64-byte row chosen by slot = l >> 2; the parity (bank half) of each slot's
// row follows a pattern.  ncu's l1tex wavefront counters tell how the hardware
// groups lanes into phases.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(const int* __restrict__ rows, float* out, int iters) {
    __shared__ float4 lut[256 * 4];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) lut[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int row = rows[lane >> 2];
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v = lut[(row + (it & 1) * 2) * 4 + (lane & 3)];
        acc += v.x + v.y + v.z + v.w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    const char* names[] = {"adjacent_pairs_01010101", "pairs_00110011", "halves_00001111",
                           "same_parity_00000000", "stride4_01230123_q", "random"};
    int pats[6][8] = {{0, 1, 2, 3, 4, 5, 6, 7}, {0, 2, 1, 3, 4, 6, 5, 7}, {0, 2, 4, 6, 1, 3, 5, 7},
                      {0, 2, 4, 6, 8, 10, 12, 14}, {0, 1, 2, 3, 4, 5, 6, 7}, {5, 9, 12, 3, 7, 7, 20, 33}};
    // rows: value*... parity of row index = bank half; pattern 0 rows 0..7 alternate parity
    int* d;
    float* o;
    cudaMalloc(&d, 32);
    cudaMalloc(&o, 1 << 20);
    for (int p = 0; p < 6; ++p) {
        int r[8];
        for (int s = 0; s < 8; ++s) r[s] = pats[p][s] * (p == 4 ? 1 : 1);
        if (p == 4) { int t[8] = {0, 1, 3, 2, 4, 5, 7, 6}; for (int s = 0; s < 8; ++s) r[s] = t[s] * 2 + (s & 1); }
        cudaMemcpy(d, r, 32, cudaMemcpyHostToDevice);
        probe<<<1, 32>>>(d, o, 1000);
        cudaDeviceSynchronize();
        printf("%d %s\n", p, names[p]);
    }
    return 0;
}
