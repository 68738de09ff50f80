mkdir -p gpurun_out
timeout 300 python tools/step_profile.py alexconv_b128.opt.k0 40 > gpurun_out/conv_prof_alex.txt 2>&1; echo "alex $?"; head -50 gpurun_out/conv_prof_alex.txt
timeout 300 python tools/step_profile.py vggconv_b64.opt.k0 30 > gpurun_out/conv_prof_vgg.txt 2>&1; echo "vgg $?"; head -40 gpurun_out/conv_prof_vgg.txt
