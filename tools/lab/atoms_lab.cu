// atoms_lab.cu — shared-memory cost of read-and-clear (not part of the product): SM cycles per
// warp instruction (16 warps per SM, conflict-free 8-byte addresses, lane-private) for
// LDS.64, STS.64, LDS.64 + STS.64 of zero, and ATOMS.EXCH.64 (read the old value, write zero
// in one instruction), ATOMS.ADD.64 without return vs the LDS.64 + STS.64 read-modify-write —
// could SIFT clear its histogram as it reads it, and accumulate with one shared atomic?
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out, unsigned long long* cyc) {
    __shared__ unsigned long long sm[512 * 8];
    const int t = threadIdx.x;
    for (int i = t; i < 512 * 8; i += 512) sm[i] = i;
    __syncthreads();
    unsigned long long acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            unsigned long long* p = &sm[j * 512 + t];
            if (MODE == 0) acc += *(volatile unsigned long long*)p;
            if (MODE == 1) *(volatile unsigned long long*)p = acc + j;
            if (MODE == 2) { acc += *(volatile unsigned long long*)p; *(volatile unsigned long long*)p = 0ull; }
            if (MODE == 3) acc += atomicExch(p, 0ull);
            if (MODE == 4) atomicAdd(p, acc + j);   // RED.ADD.64 (result unused)
            if (MODE == 6) {  // two 32-bit atomic adds (the halves of a pair entry)
                unsigned int* q = reinterpret_cast<unsigned int*>(p);
                atomicAdd(q, (unsigned)acc + j);
                atomicAdd(q + 1, (unsigned)acc + 2 * j);
            }
            if (MODE == 5) { unsigned long long v = *(volatile unsigned long long*)p; *(volatile unsigned long long*)p = v + acc + j; }
        }
    }
    const long long t1 = clock64();
    if ((t & 31) == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (acc == 12345) out[t] = acc;
}
template <int MODE>
void run(const char* name) {
    unsigned long long *o, *c;
    cudaMalloc(&o, 512 * 8);
    cudaMalloc(&c, 8);
    cudaMemset(c, 0, 8);
    const int iters = 2000;
    k<MODE><<<148, 512>>>(iters, o, c);
    cudaDeviceSynchronize();
    cudaMemset(c, 0, 8);
    k<MODE><<<148, 512>>>(iters, o, c);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double per_warp = (double)h / (148.0 * 16);
    printf("%-22s %s SM cycles per warp-instruction-slot: %.3f\n", name, cudaGetErrorString(e), per_warp / (16.0 * iters * 8));
}
int main() {
    run<0>("LDS.64");
    run<1>("STS.64");
    run<2>("LDS.64 + STS.64 zero");
    run<3>("ATOMS.EXCH.64");
    run<4>("ATOMS.ADD.64 (no return)");
    run<5>("LDS.64 + add + STS.64");
    run<6>("2 x ATOMS.ADD.32");
    return 0;
}
