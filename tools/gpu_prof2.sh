cd $GRAFT_REPO_ROOT
# BERT-base: layer-0 GEMMs (QKV, O, FFN1, FFN2 = cluster split-K), attention (mma), LayerNorm
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -c 4 -o gpurun_out/prof_gemm_bert_r1c python tools/profile_target.py bert-base 0 > gpurun_out/ncu_g.log 2>&1; echo gemm rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_attention_mma|k_layernorm" -c 3 -o gpurun_out/prof_attn_ln_r1c python tools/profile_target.py bert-base 0 > gpurun_out/ncu_a.log 2>&1; echo attn rc=$?
# GPT-2 (2 layers, XL widths): the proj2 GEMM (K = 6400) runs cluster split-K
timeout 900 ncu --set full --clock-control none -k regex:k_gemm -c 4 -o gpurun_out/prof_gemm_gpt_r1c python tools/profile_target.py gpt2-2L 0 > gpurun_out/ncu_g2.log 2>&1; echo gemm2 rc=$?
