// Standalone timing of the tcgen05 GEMM kernel over (BN, split-K) for the batch-1 shapes of the
// paper's models (tools only; feeds the cost model of runtime.cpp: choose_tiling).
// Back-to-back PDL launches timed with CUDA events, like consecutive layers of an invoke graph.
#ifdef PHASES
#define FSW_GEMM_TIMING 1
#endif
#include "../paper_2306_03622_b200/csrc/gemm_tc.cu"
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <cmath>
#include <vector>
using namespace fsw;

int main(int argc, char** argv) {
    // optional: gemm_bench <shape-name> <bn> <splits>  -> only that config (for ncu)
    const char* only = argc > 1 ? argv[1] : nullptr;
    const int only_bn = argc > 2 ? atoi(argv[2]) : 0;
    const uint32_t only_s = argc > 3 ? (uint32_t)atoi(argv[3]) : 0;
    const uint32_t only_mc = argc > 4 ? (uint32_t)atoi(argv[4]) : 0;
    struct Shape { const char* name; uint32_t M, K, N; };
    Shape shapes[] = {{"bert.qkv", 128, 768, 2304}, {"bert.o", 128, 768, 768}, {"bert.ffn1", 128, 768, 3072},
                      {"bert.ffn2", 128, 3072, 768}, {"gpt.qkv", 128, 1600, 4800}, {"gpt.fc", 128, 1600, 6400},
                      {"gpt.proj2", 128, 6400, 1600}, {"rn.s1.1x1", 3136, 64, 64}, {"rn.s1.exp", 3136, 64, 256},
                      {"rn.s3.1x1", 196, 1024, 256}, {"rn.s3.exp", 196, 256, 1024}, {"rn.s4.1x1", 49, 2048, 512},
                      {"rn.s4.exp", 49, 512, 2048}, {"rn.s4.3x3(im2col)", 49, 4608, 512}};
    init_gemm_attrs();
    uint8_t *A, *W, *O;
    float* part;
    uint32_t* ctr;
    cudaMalloc(&A, 64 << 20); cudaMalloc(&W, 64 << 20); cudaMalloc(&O, 64 << 20);
    cudaMalloc(&part, 64 << 20); cudaMalloc(&ctr, 1 << 20); cudaMemset(ctr, 0, 1 << 20);
    {  // random bf16 in [-1, 1): outputs of different tilings are compared against each other
        std::vector<uint16_t> hv((64 << 20) / 2);
        uint32_t x = 12345;
        for (auto& v : hv) { x = x * 1664525u + 1013904223u; float f = ((x >> 8) * (1.0f / 16777216.0f)) * 2.0f - 1.0f;
                             uint32_t u; memcpy(&u, &f, 4); v = (uint16_t)(u >> 16); }
        cudaMemcpy(A, hv.data(), 64 << 20, cudaMemcpyHostToDevice);
        for (auto& v : hv) { x = x * 1664525u + 1013904223u; float f = ((x >> 8) * (1.0f / 16777216.0f)) * 0.1f - 0.05f;
                             uint32_t u; memcpy(&u, &f, 4); v = (uint16_t)(u >> 16); }
        cudaMemcpy(W, hv.data(), 64 << 20, cudaMemcpyHostToDevice);
    }
    std::vector<uint16_t> ref, got;
    DevDesc* dd; cudaMalloc(&dd, sizeof(DevDesc));
    DevDesc h{W, W, 0, 0}; cudaMemcpy(dd, &h, sizeof h, cudaMemcpyHostToDevice);
    DevCtl* ctl; cudaMalloc(&ctl, sizeof(DevCtl)); cudaMemset(ctl, 0, sizeof(DevCtl));
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (auto& sh : shapes) {
        if (only && strcmp(only, sh.name)) continue;
        const uint32_t n_pad = (sh.N + 15) / 16 * 16, kt = sh.K / 64;
        double best = 1e9; int bb = 0; uint32_t bs = 0, bm = 1, bz = 0, bmr = 128, bsab = 0;
        ref.clear();
        {
        const uint32_t sab = 0;  // the swap-AB variant measured in profiles/r01/gemm_swap_ab_sweep.txt was not kept
        for (int bn : {16, 32, 64, 128}) {
            if (n_pad % bn || (only_bn && bn != only_bn)) continue;
            for (uint32_t mc : {1u, 2u, 4u, 8u}) {
            if ((n_pad / bn) % mc || (only_mc && mc != only_mc)) continue;
            for (uint32_t S : {1u, 2u, 3u, 4u, 6u, 8u, 12u, 16u, 24u, 36u}) {
            for (uint32_t cl : {0u, 1u}) {  // split-K reduction: global partials (0) / cluster DSMEM (1)
            for (uint32_t mr : {128u, 64u}) {  // activation rows per M tile
                if (S > kt || (only_s && S != only_s)) continue;
                if (ref.empty() && (sab || bn != 32 || S != 1 || mc != 1 || cl || mr != 128)) {
                    // reference output of this shape: BN = 32, no split, no swap-AB
                    CUtensorMap tr; make_tmap_act(&tr, A, sh.M, sh.K, sh.K, 128);
                    GemmArgs r{}; r.M = sh.M; r.N = sh.N; r.K = sh.K; r.n_pad = n_pad; r.has_bias = 1; r.out = O; r.out_bf16 = 1;
                    r.ld_out = sh.N; r.bn = n_pad % 32 ? 16 : 32; r.m_rows = 128; r.splits = 1; r.kt_per = kt; r.part = part; r.ctr = ctr; r.mc = 1;
                    Wait w0{}; w0.ctl = ctl;
                    launch_gemm(s, dd, w0, &tr, r);
                    cudaStreamSynchronize(s);
                    ref.resize((size_t)sh.M * sh.N);
                    cudaMemcpy(ref.data(), O, ref.size() * 2, cudaMemcpyDeviceToHost);
                }
                if (cl && (S < 2 || S > 8 || mc > 1)) continue;
                if (getenv("CZ_ONLY") && !cl && S > 1) continue;
                if (getenv("NO_MC") && mc > 1) continue;
                const uint32_t kt_per = (kt + S - 1) / S;
                if ((kt + kt_per - 1) / kt_per != S) continue;
                if (mr == 64 && mc > 1) continue;
                if (getenv("MR") && (uint32_t)atoi(getenv("MR")) != mr) continue;
                const uint32_t ctas = ((sh.M + mr - 1) / mr) * (n_pad / bn) * S;
                if (ctas > 600) continue;
                CUtensorMap tm;
                if (!make_tmap_act(&tm, A, sh.M, sh.K, sh.K, mr < 128 ? mr : 128 / mc)) { printf("tmap fail\n"); return 1; }
                GemmArgs a{}; a.M = sh.M; a.N = sh.N; a.K = sh.K; a.n_pad = n_pad; a.w_off = 0; a.b_off = 0;
                a.has_bias = 1; a.act = 0; a.res = nullptr; a.out = O; a.out_bf16 = 1; a.ld_out = sh.N; a.bn = bn;
                a.m_rows = mr; a.splits = S; a.kt_per = kt_per; a.part = part; a.ctr = ctr; a.mc = mc; a.cz = cl ? S : 0;
                Wait w{}; w.ctl = ctl;
                for (int i = 0; i < 3; ++i) launch_gemm(s, dd, w, &tm, a);
                cudaEventRecord(e0, s);
                const int reps = 50;
                for (int i = 0; i < reps; ++i) launch_gemm(s, dd, w, &tm, a);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                const double us = ms * 1000 / reps;
                const double wbytes = 2.0 * n_pad * sh.K;
                double err = 0, mref = 0;
                if (!ref.empty()) {
                    got.resize(ref.size());
                    cudaMemcpy(got.data(), O, got.size() * 2, cudaMemcpyDeviceToHost);
                    auto f = [](uint16_t v) { uint32_t u = (uint32_t)v << 16; float x; memcpy(&x, &u, 4); return (double)x; };
                    for (size_t i = 0; i < ref.size(); ++i) { err = std::max(err, std::fabs(f(got[i]) - f(ref[i]))); mref = std::max(mref, std::fabs(f(ref[i]))); }
                }
                printf("%-18s M=%5u K=%5u N=%5u BN=%3d S=%2u%s mc=%u mr=%3u%s ctas=%4u: %7.2f us  (W %.0f GB/s, %.1f TF/s) err %.1e\n", sh.name, sh.M,
                       sh.K, sh.N, bn, S, cl ? "c" : " ", mc, mr, sab ? " sab" : "", ctas, us, wbytes / us / 1e3,
                       2.0 * sh.M * sh.N * sh.K / us / 1e6, mref > 0 ? err / mref : -1.0);
                if (us < best) { best = us; bb = bn; bs = S; bm = mc; bz = cl; bmr = mr; bsab = sab; }
#ifdef PHASES
                // one isolated launch: per-CTA %globaltimer stamps -> mean phase durations
                cudaDeviceSynchronize();
                launch_gemm(s, dd, w, &tm, a);
                cudaDeviceSynchronize();
                static unsigned long long st[1024][6];
                cudaMemcpyFromSymbol(st, g_gemm_stamp, sizeof st);
                uint32_t nct = ctas > 1024 ? 1024 : ctas;
                unsigned long long t0 = ~0ull, t1 = 0;
                double ph[5] = {0};
                uint32_t nfull = 0;
                for (uint32_t c = 0; c < nct; ++c) {
                    t0 = std::min(t0, st[c][0]);
                    t1 = std::max(t1, st[c][5]);
                    if (st[c][5] == 0) continue;  // split-K CTAs that were not last skip stamp 5
                    ++nfull;
                    for (int p = 0; p < 5; ++p) ph[p] += (double)(st[c][p + 1] - st[c][p]);
                }
                if (nfull)
                    printf("    phases (us, mean over %u CTAs): setup %.2f  mainloop-issue %.2f  mma-done %.2f  tmem->smem %.2f  epilogue %.2f  | span %.2f\n",
                           nfull, ph[0] / nfull / 1e3, ph[1] / nfull / 1e3, ph[2] / nfull / 1e3, ph[3] / nfull / 1e3,
                           ph[4] / nfull / 1e3, (t1 - t0) / 1e3);
#endif
            }
            }
            }
            }
        }
        }
        printf("  BEST %-18s BN=%d S=%u%s mc=%u mr=%u%s %.2f us\n", sh.name, bb, bs, bz ? "c" : "", bm, bmr, bsab ? " sab" : "", best);
    }
    cudaError_t e = cudaGetLastError();
    printf("last error: %s\n", cudaGetErrorString(e));
    return 0;
}
