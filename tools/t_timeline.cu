// CTA timeline of one steady-state 1080p Q=8 step (default schedule) (fit -> blur+solve -> apply, PDL chain,
// replayed from a CUDA graph over a rotating pool of 4 frames): globaltimer stamps at CTA
// entry, past the grid-dependency wait, and exit (FLR_TL in flr_pipe.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFLR_TIMELINE -DFLR_Q=8 \
//        -Iinclude -lcuda tools/t_timeline.cu -o tools/t_timeline
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>
#include "../paper_2410_11625_b200/csrc/flr_inst.cu"
using namespace flr;

int main(int argc, char** argv)
{
    constexpr int Q = 8, D = 8, NP = 4;
    const int W = 1920, H = 1080, Bx = W / D, By = (H + D - 1) / D;
    const size_t plane = (size_t)W * H;
    std::vector<float*> G(NP), Y(NP), O(NP);
    std::vector<float> hg(plane * Q), hy(plane * 3);
    for (size_t i = 0; i < hg.size(); ++i) hg[i] = 0.5f + 0.25f * std::sin(0.001f * (float)i);
    for (size_t i = 0; i < hy.size(); ++i) hy[i] = 0.3f + 0.2f * std::cos(0.0007f * (float)i);
    for (int k = 0; k < NP; ++k) {
        cudaMalloc(&G[k], plane * Q * 4);
        cudaMalloc(&Y[k], plane * 3 * 4);
        cudaMalloc(&O[k], plane * 3 * 4);
        cudaMemcpy(G[k], hg.data(), hg.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(Y[k], hy.data(), hy.size() * 4, cudaMemcpyHostToDevice);
    }
    double *mom, *hb;
    float *raw, *models;
    cudaMalloc(&mom, (size_t)mom_pitch(Bx) * By * Dims<Q>::KM * 8);
    cudaMalloc(&hb, (size_t)mom_pitch(Bx) * By * Dims<Q>::KM * 8);
    cudaMalloc(&raw, 16);
    cudaMalloc(&models, (size_t)Bx * By * Dims<Q>::MSTRIDE * 4);
    Taps t{};
    t.R = 3;
    for (int i = -3; i <= 3; ++i) t.g[3 + i] = std::exp(-(double)(i * i) / (2.0 * 1.25 * 1.25));
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto has = [&](const char* a) {
        for (int i = 1; i < argc; ++i)
            if (std::string(argv[i]) == a) return true;
        return false;
    };
    const bool noapply = has("noapply");  // fit + K2 only
    const bool early = has("early");
    const std::string mode = std::string(noapply ? "staged (no apply)" : "staged") + (early ? ", inputs ready" : "");
    auto step = [&](int k) {
        LaunchCtx ctx;
        ctx.s = s;
        ctx.keep_guides = !noapply;  // as flr_denoise: the apply re-reads the fit's guides
        ctx.early = early;           // FLR_FLAG_INPUTS_READY (argument "early")
        launch_fit<Q>(1, W, H, D, Bx, By, G[k], Y[k], raw, mom, hb, models, Dims<Q>::MSTRIDE, 1e-5, 1e-4, t, ctx);
        if (!noapply) launch_apply<Q>(1, W, H, D, Bx, By, models, Dims<Q>::MSTRIDE, G[k], O[k], ctx);
    };
    for (int i = 0; i < 20; ++i) step(i % NP);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < NP; ++k) step(k);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 500; ++r) cudaGraphLaunch(ge, s);  // clocks up
    cudaEventRecord(e0, s);
    for (int r = 0; r < 200; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: graph step %.2f us (%s)\n", mode.c_str(), 1e3 * ms / (200 * NP), cudaGetErrorString(cudaGetLastError()));
    std::vector<long long> tl(3 * 1024 * 4);
    cudaMemcpyFromSymbol(tl.data(), flr::g_flr_tl, tl.size() * 8);
    const int ncta[3] = {148, ((Bx + 31) / 32) * ((By + 7) / 8), 148};
    long long t0 = tl[0];
    for (int c = 0; c < ncta[0]; ++c) t0 = std::min(t0, tl[c * 4]);
    const char* nm[3] = {"fit", "k2", "apply"};
    for (int k = 0; k < 3; ++k) {
        long long emin = 1LL << 62, emax = 0, wmin = 1LL << 62, wmax = 0, xmin = 1LL << 62, xmax = 0;
        double dur = 0;
        for (int c = 0; c < ncta[k]; ++c) {
            const long long* q = &tl[(k * 1024 + c) * 4];
            emin = std::min(emin, q[0]), emax = std::max(emax, q[0]);
            wmin = std::min(wmin, q[1]), wmax = std::max(wmax, q[1]);
            xmin = std::min(xmin, q[2]), xmax = std::max(xmax, q[2]);
            dur += q[2] - std::max(q[0], q[1]);
        }
        printf("%-5s ctas %3d  entry %6.2f..%6.2f  wait-passed %6.2f..%6.2f  exit %6.2f..%6.2f  mean busy %5.2f us\n",
               nm[k], ncta[k], (emin - t0) * 1e-3, (emax - t0) * 1e-3, (wmin - t0) * 1e-3, (wmax - t0) * 1e-3,
               (xmin - t0) * 1e-3, (xmax - t0) * 1e-3, dur / ncta[k] * 1e-3);
        std::vector<double> xs;
        for (int c = 0; c < ncta[k]; ++c) xs.push_back((tl[(k * 1024 + c) * 4 + 2] - t0) * 1e-3);
        std::sort(xs.begin(), xs.end());
        printf("      exit deciles:");
        for (int d = 0; d <= 10; ++d) printf(" %.1f", xs[std::min((int)xs.size() - 1, d * (int)xs.size() / 10)]);
        printf("\n");
    }
    if (has("cta")) {  // fit: per-CTA exit (relative), SM id, items
        std::vector<std::pair<long long, int>> ex;
        for (int c = 0; c < ncta[0]; ++c) ex.push_back({tl[c * 4 + 2] - t0, c});
        std::sort(ex.begin(), ex.end());
        printf("fit CTA exits (us: cta/sm):");
        for (auto& e : ex) printf(" %.1f:%d/%lld", e.first * 1e-3, e.second, tl[e.second * 4 + 3]);
        printf("\n");
    }
    return 0;
}
