import sys, ctypes
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N
g = gd.Graph(4, np.asarray([[0, 1], [1, 2], [0, 2], [2, 3]]))
tab = np.ascontiguousarray(gd.micro_table(g))
print("table ok", tab.shape, flush=True)
L = N.lib()
h = ctypes.c_void_p(); bad = ctypes.c_int64(-1)
orig = np.ascontiguousarray(g.orig_ids, dtype=np.int64)
rc = L.gd_micro_csv(g.handle, N.vptr(tab), 0, N.vptr(orig), ctypes.byref(h), ctypes.byref(bad))
print("rc", rc, "bad", bad.value, "h", h.value, flush=True)
size = L.gd_text_size(h)
print("size", size, flush=True)
buf = bytearray(size)
view = (ctypes.c_char * size).from_buffer(buf)
rc = L.gd_text_copy(h, 0, size, view)
print("copy rc", rc, bytes(buf[:200]), flush=True)
del view
L.gd_text_free(h)
print("freed", flush=True)
