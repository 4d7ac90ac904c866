python -m pytest tests/test_gpu_attention.py tests/test_gpu_c2.py -m gpu -q > gpurun_out/pt_mask.txt 2>&1
for r in 1 2; do for x in "" build/variants/oldattn.so; do FQ_LIB=$x python scripts/masked_generate_ab.py >> gpurun_out/mask_ab.txt 2>&1; done; done
