import sys, runpy
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
K._lib = K.load_library(sys.argv[1])
runpy.run_path('scratch/attn_bench.py', run_name='__main__')
