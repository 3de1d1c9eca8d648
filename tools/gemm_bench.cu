// Standalone timing of the tcgen05 GEMM kernel (tools only): back-to-back launches with CUDA
// events, plus per-CTA %globaltimer phase stamps (FSW_GEMM_TIMING).
#define FSW_GEMM_TIMING 1
#include "../paper_2306_03622_b200/csrc/gemm_tc.cu"
#include <cstdio>
#include <vector>
using namespace fsw;

int main() {
    struct Shape { const char* name; uint32_t M, K, N; };
    Shape shapes[] = {{"bert.qkv", 128, 768, 2304}, {"bert.o", 128, 768, 768}, {"bert.ffn1", 128, 768, 3072},
                      {"bert.ffn2", 128, 3072, 768}, {"gpt.fc", 128, 1600, 6400}, {"gpt.proj2", 128, 6400, 1600},
                      {"rn.conv1", 12544, 192, 64}, {"rn.s1.3x3", 3136, 576, 64}, {"rn.s4.3x3", 49, 4608, 512},
                      {"rn.s4.exp", 49, 512, 2048}};
    init_gemm_attrs();
    uint8_t *A, *W, *O;
    cudaMalloc(&A, 64 << 20); cudaMalloc(&W, 64 << 20); cudaMalloc(&O, 64 << 20);
    cudaMemset(A, 0x3c, 64 << 20); cudaMemset(W, 0x3c, 64 << 20);
    DevDesc* dd; cudaMalloc(&dd, sizeof(DevDesc));
    DevDesc h{W, 0}; cudaMemcpy(dd, &h, sizeof h, cudaMemcpyHostToDevice);
    DevCtl* ctl; cudaMalloc(&ctl, sizeof(DevCtl)); cudaMemset(ctl, 0, sizeof(DevCtl));
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode : {0}) {
    for (auto& sh : shapes) {
        for (int bn : {16, 32, 64, 128}) {
            uint32_t n_pad = (sh.N + 15) / 16 * 16;
            if (n_pad % bn) continue;
            CUtensorMap tm;
            if (!make_tmap_act(&tm, A, sh.M, sh.K, sh.K)) { printf("tmap fail\n"); return 1; }
            GemmArgs a{}; a.M = sh.M; a.N = sh.N; a.K = sh.K; a.n_pad = n_pad; a.w_off = 0; a.b_off = 0;
            a.has_bias = 1; a.act = 0; a.res = nullptr; a.out = O; a.out_bf16 = 1; a.ld_out = sh.N; a.bn = bn;
            Wait w{nullptr, 0, ctl, 0};
            for (int i = 0; i < 3; ++i) launch_gemm(s, dd, w, &tm, a);
            cudaEventRecord(e0, s);
            const int reps = 20;
            for (int i = 0; i < reps; ++i) launch_gemm(s, dd, w, &tm, a);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            // single launch stamps
            cudaMemsetAsync(O, 0, 1, s);
            launch_gemm(s, dd, w, &tm, a);
            cudaStreamSynchronize(s);
            static unsigned long long st[1024][6];
            cudaMemcpyFromSymbol(st, g_gemm_stamp, sizeof st);
            uint32_t nct = ((sh.M + 127) / 128) * (n_pad / bn); if (nct > 1024) nct = 1024;
            unsigned long long t0 = ~0ull, tend = 0; double ph[5] = {0};
            for (uint32_t c = 0; c < nct; ++c) { t0 = std::min(t0, st[c][0]); tend = std::max(tend, st[c][5]); for (int p = 0; p < 5; ++p) ph[p] += (double)(st[c][p + 1] - st[c][p]); }
            double flops = 2.0 * sh.M * sh.N * sh.K;
            printf("%-10s M=%5u K=%5u N=%5u BN=%3d ctas=%4u: %7.2f us/launch (%.1f TF/s)  span=%.2f us  phases(us): setup %.2f mainloop %.2f (+%.2f) tmem->smem %.2f store %.2f\n",
                   sh.name, sh.M, sh.K, sh.N, bn, nct, ms * 1000 / reps, flops / (ms / reps * 1e-3) / 1e12, (tend - t0) / 1e3,
                   ph[0] / nct / 1e3, ph[1] / nct / 1e3, ph[2] / nct / 1e3, ph[3] / nct / 1e3, ph[4] / nct / 1e3);
        }
    }
    }
    cudaError_t e = cudaGetLastError();
    printf("last error: %s\n", cudaGetErrorString(e));
    return 0;
}
