timeout 300 python tools/step_profile.py alexconv_b128.opt.k0 40 | grep -v "gemm  gemm\|col2im  " 
timeout 300 python tools/step_profile.py vggconv_b64.opt.k0 6 | head -5
