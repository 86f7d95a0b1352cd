for v in 0 1; do
  cp scratch/variants/libgalv_mc$v.so paper_2504_21411_b200/libgalv_b200.so
  echo "multicast=$v"; timeout 200 python scratch/attn_long.py
done
