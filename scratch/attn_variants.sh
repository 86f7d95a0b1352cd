for v in 2 3 4; do
  cp scratch/variants/libgalv_v$v.so paper_2504_21411_b200/libgalv_b200.so
  echo "poly every $v:"; timeout 120 python scratch/attn_bench.py
done
