# Test the tests: build one deliberately broken library per CY_MUTANT value and run the GPU tests
# that should catch it (conftest loads the library named by CY_ATTN_EXPERIMENTS_LIB for the whole
# session).  Every line must end in "caught".  GPU box: bash scripts/mutants.sh
set -u
run() {  # mutant id, pytest -k expression
  [ -f build/exp/libcypress_mutant$1.so ] || python scripts/build_experiment.py mutant$1 CY_MUTANT=$1 > /dev/null 2>&1 \
    || { echo "mutant $1: build failed"; return; }
  out=$(CY_ATTN_EXPERIMENTS_LIB=build/exp/libcypress_mutant$1.so timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q -k "$2" 2>&1 | tail -1)
  case "$out" in *failed*) echo "mutant $1 ($2): caught -- $out";; *) echo "mutant $1 ($2): NOT caught -- $out";; esac
  rm -f build/exp/libcypress_mutant$1.so
}
run 1 "alpha_beta or beta_c or dual_pair or batched_64x1024_beta"
run 2 "splitk"
run 3 "rowreduce"
run 4 "attention and not variants"
run 5 "integer_bit_exact or identity or full_8192"
