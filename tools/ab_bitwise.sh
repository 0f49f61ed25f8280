# Run a dump script with the in-tree library and with a variant, compare bitwise.
# usage: bash tools/ab_bitwise.sh tools/<dump>.py tools/variants/<lib>.so
DIVUQ_LIB_PATH=$2 python $1 gpurun_out/abA.npz && python $1 gpurun_out/abB.npz && python -c "
import numpy as np
a = np.load('gpurun_out/abA.npz'); b = np.load('gpurun_out/abB.npz')
for k in a.files:
    x, y = a[k], b[k]
    u = np.uint64 if x.dtype.itemsize == 8 else np.uint32
    same = np.array_equal(x.view(u), y.view(u))
    print(k, 'bitwise' if same else 'DIFF max %.3g n=%d' % (np.nanmax(np.abs(x - y)), (x.view(u) != y.view(u)).sum()))
"
