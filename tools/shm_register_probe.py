"""Which /dev/shm mapping sizes can cudaHostRegister pin on this box?"""
import ctypes, mmap, os, resource, sys
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L
print("RLIMIT_MEMLOCK", resource.getrlimit(resource.RLIMIT_MEMLOCK), flush=True)
for gb in (0.25, 1, 4, 8, 17):
    n = int(gb * (1 << 30))
    path = f"/dev/shm/pshard_probe_{os.getpid()}"
    fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o600)
    os.ftruncate(fd, n)
    mm = mmap.mmap(fd, n)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    for flags in (1, 0):
        try:
            L.call("ps_host_register", addr, n, flags)
            print(gb, "GB register ok (portable=%d)" % flags, flush=True)
            L.call("ps_host_unregister", addr)
        except Exception as e:
            print(gb, "GB register FAILED (portable=%d):" % flags, str(e)[:120], flush=True)
    # touch pages first then retry
    try:
        ctypes.memset(addr, 0, n)
        L.call("ps_host_register", addr, n, 1)
        print(gb, "GB register after touching ok", flush=True)
        L.call("ps_host_unregister", addr)
    except Exception as e:
        print(gb, "GB register after touching FAILED:", str(e)[:120], flush=True)
    mm.close(); os.close(fd); os.unlink(path)
