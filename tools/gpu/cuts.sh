timeout 600 python tools/nshapes_knobs.py base 2>&1
for st in alexconv_b128.opt.k0 vggconv_b64.opt.k0; do
  for kn in "" "30:5" ""; do
    echo "== $st knobs=$kn"; TPX_GEMM_KNOBS=$kn timeout 300 python tools/step_profile.py $st 0 2>&1 | head -2 | tail -1
  done
done
timeout 600 python tools/nshapes_probe.py 2>&1 | grep -v "^{" > gpurun_out/r2_nshapes_v2.txt; cat gpurun_out/r2_nshapes_v2.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/cuts_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/cuts_pytest.log
