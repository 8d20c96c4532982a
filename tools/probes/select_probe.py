import ctypes as C
import numpy as np
import torch
from paper_1612_06457_b200 import _lib
from paper_1612_06457_b200 import device as dev

L = _lib.lib()
for n in (100, 1517, 1000):
    for dtype in (np.float64, np.float32):
        x = np.linspace(0.0, 1.0, n).astype(dtype)
        t = torch.from_numpy(x).cuda()
        out = torch.empty(2, dtype=torch.float64, device="cuda")
        ws = dev.workspace("plane_select", L.ut_plane_select_ws(), t.device)
        for r0, r1 in ((1, 95), (5, 95), (1, n), (n, 1)):
            ranks = (C.c_int64 * 2)(r0, r1)
            _lib.check(L.ut_plane_select(t.data_ptr(), _lib.UT_F32 if dtype == np.float32 else _lib.UT_F64,
                                         n, ranks, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                         dev.stream_handle()), "s")
            s = np.sort(x)
            print(n, dtype.__name__, (r0, r1), out.cpu().numpy(), (s[r0 - 1], s[r1 - 1]))
