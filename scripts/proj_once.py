import sys; sys.path.insert(0,'.')
from paper_1602_00138_b200 import romdot as R
print(R.bench_projection(2097152, 69, True, 3))
