S="256,256,64,30,148 768,768,64,30,64 1536,1536,64,40,32"
for v in "X=1" "CBIE_PCHOL_W=1" "CBIE_PCHOL_W=2" "CBIE_PCHOL_W=4" "CBIE_PCHOLH_W=1" "CBIE_PCHOLH_W=4" "CBIE_PCHOLH_W=8" "CBIE_JACOBI_T=128" "CBIE_JACOBI_T=256"; do
  echo "== $v"; env $v python tools/trunc_bench.py $S
done
