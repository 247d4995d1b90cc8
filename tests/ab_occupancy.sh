for cfg in "1 4" "1 3" "1 2" "0 2"; do set -- $cfg; echo "HALF=$1 CTAS=$2"; TPMG_JACOBI_HALF=$1 TPMG_JACOBI_CTAS=$2 TPMG_ROUNDS=3 python tests/ab_kernels.py jacobi post rupdate jacobi0; done
