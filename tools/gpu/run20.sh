set -x; mkdir -p gpurun_out
for c in alexnet_b128 vgg_b64 cfg5_mlp3x32768_b32 alexfc_b128 vggfc_b64 cfg1_mlp3x1024_b64; do
  timeout 900 python bench.py --config $c > gpurun_out/r2_bench_$c.log 2>&1; echo "$c exit $?"; tail -1 gpurun_out/r2_bench_$c.log | cut -c1-200
done
timeout 900 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/r2_bench_bf16.log 2>&1; echo "bf16 exit $?"; tail -1 gpurun_out/r2_bench_bf16.log | cut -c1-200
