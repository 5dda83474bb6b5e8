import ctypes as C, os, torch
torch.cuda.init()
lib = C.CDLL(os.path.join(os.path.dirname(__file__), "..", "tests", "cuda", "libtcprobe.so"))
lib.tc_timing.restype = C.c_longlong
for mode, name in [(0, "SS M128 N=32"), (1, "TS M128 N=16"), (2, "SS N=32 2acc"), (3, "SS M128 N=256"), (4, "SS M64 N256"), (5, "SS M64 N128"), (6, "SS M128 N128"), (7, "SS M64 N64"), (8, "SS M128 N64"), (9, "SS M64 N32"), (10, "UNROLLED SS M128 N32"), (11, "UNROLLED SS M128 N256"), (12, "UNROLLED TS M128 N16"), (13, "UNROLLED SS M64 N256"), (14, "UNROLLED SS M64 N192"), (15, "UNROLLED SS M64 N128"), (16, "BF16 TS N64+N32 no commit"), (17, "BF16 TS N64+N32 commit/4"), (19, "BF16 TS N32+N32 no commit")]:
    res = []
    for n in (1, 8, 128, 512):
        lib.tc_timing(mode, n)
        res.append((n, min(lib.tc_timing(mode, n) for _ in range(5))))
    print(name, res, flush=True)

import numpy as np
fp = C.POINTER(C.c_float)
A = np.arange(64 * 32, dtype=np.float32).reshape(64, 32) % 7
A = (A + np.arange(64)[:, None] * 0).astype(np.float32)
A = np.zeros((64, 32), np.float32); A[np.arange(64), 0] = np.arange(64) + 1   # row i -> value i+1 in col 0
B = np.zeros((32, 32), np.float32); B[:, 0] = 1.0; B[np.arange(32), 1] = 1.0
dump = np.zeros((128, 32), np.float32)
rc = lib.tc_m64(A.ctypes.data_as(fp), B.ctypes.data_as(fp), dump.ctypes.data_as(fp))
print("m64 rc", rc)
for lane in range(128):
    print("lane", lane, dump[lane, :4].tolist())
X = (np.arange(40 * 64, dtype=np.float32)).reshape(40, 64)
rows = np.array([5, 17, 3, 39], dtype=np.int32)
out = np.zeros(128, np.float32)
rc = lib.tc_gather4(X.ctypes.data_as(fp), 40, 64, 32, rows.ctypes.data_as(C.POINTER(C.c_int)), out.ctypes.data_as(fp))
print("gather4 rc", rc, "ok", np.array_equal(out.reshape(4, 32), X[rows, 32:64]))
