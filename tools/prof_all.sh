# ncu --set full captures of every hot kernel (one launch each, after a warm-up launch), summarised
# ON the box (the reports are too large to bring back) into gpurun_out/ncu_summary.json plus SASS
# opcode histograms of the tensor sum and the conv MAC:
#   bash tools/prof_all.sh   (kernel-name regexes match ncu's demangled form, e.g. 'k_tensor_sum<(int)1, ...>', with '.' for
#    spaces and parentheses)
NCU="ncu --set full --clock-control none --kernel-name-base demangled -f"
cap() {  # tag regex skip cmd...   (ONLY="tag ..." restricts the run)
  local tag=$1 re=$2 skip=$3; shift 3
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $tag "* ]]; then return; fi
  timeout 600 $NCU -k "regex:$re" -s $skip -c 1 -o gpurun_out/ncu_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$? $(ls -la gpurun_out/ncu_$tag.ncu-rep 2>/dev/null | awk '{print $5}')"
}
export VR_ASYNC=0 VR_MM_ORDER=5   # eager one-pass matmul_outer: the kernels the async slot graphs replay
cap ts_onepass 'k_tensor_sum_ld' 1 --import-source on python tools/step_profile.py --cfg 2 --steps 2
cap modup_ntt 'ntt_cl8<.bool.0,..int.11,.*LdLift' 1 python tools/step_profile.py --cfg 2 --steps 2
cap modup_intt 'ntt_cl8<.bool.1,..int.11,.*LdGather' 1 python tools/step_profile.py --cfg 2 --steps 2
cap ks_inner_cfg2 'k_ks_inner' 1 python tools/step_profile.py --cfg 2 --steps 2
cap moddown_store 'StRelinRescale' 1 python tools/step_profile.py --cfg 2 --steps 2
unset VR_MM_ORDER
cap ts_d01 'k_tensor_sum<.int.1,..int.512,..int.2,..int.4,..int.2>' 1 python tools/step_profile.py --cfg 2 --steps 2
cap ts_d2 'k_tensor_sum<.int.1,..int.512,..int.4,..int.4,..int.1>' 1 python tools/step_profile.py --cfg 2 --steps 2
cap ntt_cl8_fwd 'ntt_cl8<.bool.0,..int.11,.*LdPlain' 1 python tools/ntt_only.py 2
cap ntt_pass_fwd_n15 'ntt_pass<.bool.0,..bool.1,.*LdPlain' 1 python tools/ntt_only.py 4
cap ntt_pass_rows_n15 'ntt_pass<.bool.0,..bool.0,.*LdPlain,.vr::nttk::StPlain' 1 python tools/ntt_only.py 4
cap conv_mac 'k_conv_mac' 0 --import-source on python tools/step_profile.py --cfg 4 --steps 1 --images 16 --filters 16
cap ks_inner_cfg4 'k_ks_inner' 1 python tools/step_profile.py --cfg 4 --steps 1 --images 16 --filters 16
cap lift_ntt_cfg4 'ntt_pass<.bool.0,..bool.1,.*LdLift' 2 python tools/step_profile.py --cfg 4 --steps 1 --images 16 --filters 16
cap pt_matvec 'k_pt_matvec' 2 python tools/cfg3_profile.py
cap enc_ntt 'LdSymEnc' 1 python tools/e2e_profile.py
cap encode 'k_encode' 1 python tools/e2e_profile.py
cap decode 'k_decode' 1 python tools/e2e_profile.py
unset VR_ASYNC
cap ts_cfg5a 'k_tensor_sum' 1 python tools/cfg5a_prof.py
cap ts_many_cfg1 'k_tensor_sum_ld<.int.1,' 1 python tools/many_probe.py 1 32

python tools/ncu_summarize.py gpurun_out gpurun_out/ncu_summary.json > gpurun_out/ncu_summarize.log 2>&1; echo "summary rc=$?"
for t in ts_onepass conv_mac; do
  ncu -i gpurun_out/ncu_$t.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$t.csv 2>/dev/null
  python tools/sass_hist.py gpurun_out/sass_$t.csv > gpurun_out/sass_hist_$t.txt 2>&1; echo "sass $t rc=$?"
  rm -f gpurun_out/sass_$t.csv
done
rm -f gpurun_out/*.ncu-rep
