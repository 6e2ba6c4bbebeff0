// Standalone check of k_blur_solve (TMA halo) on a small moment field, with error checks.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_tiles.cuh"

using namespace flr;
namespace flr {
__device__ long long g_flr_dbg_times[64];
}
#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));    \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

int probe(int Bx, int By, int planes, int bx, int by, int bz, int x, int y, int z, CUtensorMapDataType dt, int es);
__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int bx, int by, int bz, int x, int y, int z, double* out, int es);
int main(int argc, char** argv)
{
    if (argc > 3) {
        const int v = atoi(argv[3]);
        const CUtensorMapDataType f64 = CU_TENSOR_MAP_DATA_TYPE_FLOAT64, f32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        if (v == 0) return probe(240, 135, 72, 38, 10, 12, 0, 0, 0, f64, 8);
        if (v == 1) return probe(240, 135, 72, 38, 10, 12, 0, 0, 0, f32, 4);
        if (v == 2) return probe(240, 135, 72, 32, 8, 1, 0, 0, 0, f64, 8);
        if (v == 3) return probe(240, 135, 72, 38, 10, 12, -3, -3, 0, f64, 8);
        if (v == 4) return probe(240, 135, 72, 38, 1, 1, 0, 0, 0, f64, 8);
        if (v == 5) return probe(240, 135, 72, 16, 10, 12, 0, 0, 0, f64, 8);
        if (v == 6) return probe(240, 135, 72, 32, 10, 12, 0, 0, 0, f64, 8);
        if (v == 7) return probe(240, 135, 72, 38, 1, 1, -3, 0, 0, f64, 8);
        if (v == 8) return probe(240, 135, 72, 38, 10, 1, 0, -3, 0, f64, 8);
        if (v == 9) return probe(240, 135, 72, 38, 10, 12, -4, 0, 0, f64, 8);
        if (v == 10) return probe(240, 135, 72, 38, 10, 12, -2, 0, 0, f64, 8);
        if (v == 11) return probe(240, 135, 72, 38, 10, 12, -3, 0, 0, f32, 4);
        if (v == 12) return probe(240, 135, 72, 38, 10, 12, -2, 0, 0, f32, 4);
        return 0;
    }
    constexpr int Q = 8, R = 3;
    const int Bx = argc > 1 ? atoi(argv[1]) : 8, By = argc > 2 ? atoi(argv[2]) : 8, n = 1;
    const int Bxp = mom_pitch(Bx), KM = Dims<Q>::KM;
    std::vector<double> h((size_t)n * KM * By * Bxp, 0.0);
    for (int k = 0; k < KM; ++k)
        for (int y = 0; y < By; ++y)
            for (int x = 0; x < Bx; ++x) h[((size_t)k * By + y) * Bxp + x] = (k == 0 ? 64.0 : 1.0 + 0.01 * (k + x + y));
    double* mom;
    float* models;
    CK(cudaMalloc(&mom, h.size() * 8));
    CK(cudaMalloc(&models, (size_t)Bx * By * 28 * 4));
    CK(cudaMemcpy(mom, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    bool ok = make_tmap_3d(&tm, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, n * KM, halo_x(R),
                           kTileTY + 2 * R, tile_g(R));
    printf("tmap ok=%d Bx=%d By=%d Bxp=%d\n", ok, Bx, By, Bxp);
    Taps t{};
    t.R = R;
    for (int i = -R; i <= R; ++i) t.g[R + i] = std::exp(-(double)(i * i) / (2.0 * 1.25 * 1.25));
    const size_t sm = blur_solve_smem_bytes(R);
    CK(cudaFuncSetAttribute(k_blur_solve<Q, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_blur_solve<Q, R><<<dim3(cdiv(Bx, kTileTX), cdiv(By, kTileTY), n), kTileTX * kTileTY, sm>>>(
            tm, Bx, By, models, 28, 1e-5, 1e-4, t);
        cudaEventRecord(e1);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("k_blur_solve %dx%d blocks: %.1f us\n", Bx, By, ms * 1e3);
#ifdef FLR_DBG_TIMES
    long long ht[64];
    cudaMemcpyFromSymbol(ht, g_flr_dbg_times, sizeof(ht));
    printf("tile phases (cycles from start):");
    for (int i = 0; i < ht[63]; ++i) printf(" %lld", ht[i]);
    printf("\n");
#endif
    std::vector<float> m((size_t)Bx * By * 28);
    CK(cudaMemcpy(m.data(), models, m.size() * 4, cudaMemcpyDeviceToHost));
    printf("model[0] = %g %g %g\n", m[0], m[1], m[2]);
    return 0;
}

// minimal TMA probe: one box -> smem -> global
__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int bx, int by, int bz, int x, int y, int z, double* out, int es)
{
    extern __shared__ __align__(1024) unsigned char sp[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, bx * by * bz * es);
        tma_load_3d(sp, &tm, x, y, z, &bar, policy_evict_normal());
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < bx * by * bz * es / 8; i += blockDim.x) out[i] = reinterpret_cast<double*>(sp)[i];
}

int probe(int Bx, int By, int planes, int bx, int by, int bz, int x, int y, int z, CUtensorMapDataType dt, int es)
{
    double *d, *o;
    cudaMalloc(&d, (size_t)Bx * By * planes * 8);
    cudaMalloc(&o, (size_t)bx * by * bz * 8);
    CUtensorMap tm;
    const int w = Bx * 8 / es, pitch = w;
    bool ok = make_tmap_3d(&tm, d, dt, es, w, By, pitch, planes, bx * 8 / es, by, bz);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k_probe<<<1, 128, bx * by * bz * 8>>>(tm, bx * 8 / es, by, bz, x * 8 / es, y, z, o, es);
    cudaError_t e = cudaDeviceSynchronize();
    printf("probe dt=%d box {%d,%d,%d} at (%d,%d,%d) tmap=%d -> %s\n", (int)dt, bx, by, bz, x, y, z, ok,
           cudaGetErrorString(e));
    return e != cudaSuccess;
}
