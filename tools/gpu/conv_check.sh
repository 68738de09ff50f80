timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/minb_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/minb_pytest.log
for c in alexnet_b128 vgg_b64; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/s3b_bench_$c.json 2> gpurun_out/s3b_bench_$c.err; echo "$c $?"; cut -c1-200 gpurun_out/s3b_bench_$c.json
done
timeout 300 python tools/step_profile.py alexconv_b128.opt.k0 40 > gpurun_out/r2_conv_prof_alex_v2.txt 2>&1; head -8 gpurun_out/r2_conv_prof_alex_v2.txt
