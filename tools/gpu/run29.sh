timeout 300 python tools/step_profile.py alexconv_b128.opt.k0 12
TPX_EXTRA_FLAGS=64 timeout 300 python tools/step_profile.py alexconv_b128.opt.k0 6
timeout 300 python tools/step_profile.py vggconv_b64.opt.k0 6
TPX_EXTRA_FLAGS=64 timeout 300 python tools/step_profile.py vggconv_b64.opt.k0 6
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 900 -k "conv or alex or vgg or cnn" 2>&1 | tail -3
