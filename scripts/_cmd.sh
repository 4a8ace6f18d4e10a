timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
bash scripts/ab_env.sh fused "X=0" unfused "NLD_NO_FUSED_EPILOGUE=1" fusedbc "NLD_SPREAD_BC=1"
