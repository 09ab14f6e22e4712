// bp_timing.cu — phase timestamps of bad_patch_kernel on CTA 0 (not part of the product):
// compiles the product kernel with BD_BP_TIMING and prints clock64 deltas per tile.
#define BD_BP_TIMING 1
#include "experiments/bad_patch_tensorcore_build.cu"
#include <vector>
namespace bd {
int num_sms() { int d, n; cudaGetDevice(&d); cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d); return n; }
cudaError_t ensure_smem_attr(const void* fn, int bytes) { return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
ProfScope::ProfScope(const char*, cudaStream_t) : s_(0), idx_(-1) {}
ProfScope::~ProfScope() {}
}
int main() {
    const int64_t n = 4000000;
    uint8_t* d; uint32_t* out;
    cudaMalloc(&d, n * 1024); cudaMemset(d, 7, n * 1024);
    cudaMalloc(&out, n * 32);
    bd::PatchTable tab; memset(&tab, 0, sizeof tab); tab.dp2a = 1;
    srand(3);
    for (int k = 0; k < 256; ++k) {
        for (int c = 0; c < 8; ++c) { int e = rand() % 1025; tab.t[k].off[c] = e * 132; }
        tab.t[k].m1 = 0x00f70009; tab.t[k].m2 = 0xf7000900; tab.t[k].nthr1 = -1;
    }
    for (int rep = 0; rep < 3; ++rep) bd::launch_bad_patches(d, n, tab, 256, out, nullptr, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); bd::launch_bad_patches(d, n, tab, 256, out, nullptr, 0); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    printf("kernel %.3f ms (%s)\n", ms, cudaGetErrorString(cudaGetLastError()));
    long long h[64][16];
    cudaMemcpyFromSymbol(h, bd::kern::g_bp_t, sizeof h);
    printf("tile: [start->dfull0] [->dfull1] [->built] [->barrier] [tests] [->barrier] | total | producer full-wait times rel. start (g0..g7)\n");
    for (int t = 2; t < 14; ++t) {
        long long* r = h[t];
        printf("%2d: %6lld %6lld %6lld %6lld %6lld %6lld | %6lld |", t, r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3],
               r[5] - r[4], r[6] - r[5], h[t + 1][0] - r[0]);
        printf("\n");
    }
    long long pp[64][8][4];
    cudaMemcpyFromSymbol(pp, bd::kern::g_bp_p, sizeof pp);
    printf("producer (tile 6): per group: dempty-done, full-done, issued, refill-done (rel. tile-6 compute start)\n");
    for (int g = 0; g < 2; ++g)
        printf(" g%d: %7lld %7lld %7lld %7lld\n", g, pp[6][g][0] - h[6][0], pp[6][g][1] - h[6][0], pp[6][g][2] - h[6][0],
               pp[6][g][3] - h[6][0]);
    return 0;
}
