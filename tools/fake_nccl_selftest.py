import ctypes as C, os, sys, time
import torch
lib = C.CDLL(os.environ["B2M_NCCL_LIB"])
rank, n, idfile = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
uid = (C.c_char * 128)()
if rank == 0:
    lib.ncclGetUniqueId(uid); open(idfile, "wb").write(bytes(uid))
else:
    while not os.path.exists(idfile) or os.path.getsize(idfile) < 128: time.sleep(0.01)
    uid = (C.c_char * 128).from_buffer_copy(open(idfile, "rb").read())
comm = C.c_void_p()
class U(C.Structure): _fields_ = [("internal", C.c_char * 128)]
u = U(); C.memmove(C.byref(u), uid, 128)
print(rank, "init", lib.ncclCommInitRank(C.byref(comm), n, u, rank), flush=True)
x = torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int64, device="cuda")
y = torch.zeros(2, dtype=torch.int64, device="cuda")
print(rank, "ar", lib.ncclAllReduce(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_size_t(2), 4, 0, comm, None), y.tolist(), flush=True)
