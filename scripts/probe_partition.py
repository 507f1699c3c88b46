"""Dev probe: SM counts the driver grants for green-context partitions of the B200."""
import ctypes, sys
sys.path.insert(0, ".")
import torch
from paper_2007_11831_b200 import _lib
torch.cuda.init()
for n, per in [(4, 32), (4, 36), (4, 34), (4, 37), (3, 48), (3, 49), (2, 74), (1, 148)]:
    h = ctypes.c_void_p(); act = ctypes.c_int32()
    st = _lib.lib().dbs_partition_create(n, per, ctypes.byref(h), ctypes.byref(act))
    print(n, per, "->", st, act.value, _lib.last_error() if st else "", flush=True)
