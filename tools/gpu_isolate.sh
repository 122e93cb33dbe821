for ks in 1 2 4; do
 for c in gmm_1024 gmm_256x128x256 c2d_s2; do
  echo "== $c KS=$ks"; TIR_B200_KS=$ks python tests/gpu_diag.py $c 2>&1 | grep -E "case|Error:" | head -2
 done
done
