# bench lines for every config (tag in $TAG)
mkdir -p gpurun_out
T=${TAG:-x}
timeout 900 python bench.py > gpurun_out/${T}_bench_n1.json 2> gpurun_out/${T}_bench_n1.err; echo "cfg2 $?"; cut -c1-200 gpurun_out/${T}_bench_n1.json
for c in alexnet_b128 vgg_b64 cfg5_mlp3x32768_b32; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "$c $?"; cut -c1-200 gpurun_out/${T}_bench_$c.json
done
