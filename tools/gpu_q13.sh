EKS_SPMM_PATH=grid timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_size_spmm_gram_sampled" 2>&1 | tail -30
