for v in 2 3; do
  cp scratch/variants/libgalv_nst$v.so paper_2504_21411_b200/libgalv_b200.so
  echo "dkdv NST=$v (double-buffered P/dS)"; timeout 200 python scratch/attn_bench.py; timeout 100 python -m pytest tests/test_kernels_attn.py -q -x 2>&1 | tail -1
done
