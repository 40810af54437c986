"""Two processes mapping and pinning the same /dev/shm segment at once (the replicas' path)."""
import ctypes, mmap, os, sys, time, multiprocessing as mp
sys.path.insert(0, os.getcwd())

def worker(path, n, create, q):
    from paper_2604_26334_b200.runtime import lib as L
    import torch
    torch.cuda.set_device(0)
    mode = os.environ.get("MODE", "concurrent")
    if create:
        fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o600); os.ftruncate(fd, n)
        if mode in ("fallocate", "serial"):
            os.posix_fallocate(fd, 0, n)
    else:
        while not os.path.exists(path) or os.path.getsize(path) < n: time.sleep(0.01)
        if mode == "serial":
            while not os.path.exists(path + ".pinned"): time.sleep(0.01)
        fd = os.open(path, os.O_RDWR)
    mm = mmap.mmap(fd, n)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    t0 = time.time()
    try:
        L.call("ps_host_register", addr, n, 1)
        if create: open(path + ".pinned", "w").close()
        q.put((create, "ok", round(time.time() - t0, 2)))
        time.sleep(2)
        L.call("ps_host_unregister", addr)
    except Exception as e:
        q.put((create, "FAIL " + str(e)[:100], round(time.time() - t0, 2)))

if __name__ == "__main__":
    for gb in (1, 17):
        n = gb << 30
        path = f"/dev/shm/pshard_probe2_{gb}"
        ctx = mp.get_context("spawn"); q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(path, n, c, q)) for c in (True, False)]
        [p.start() for p in ps]
        print(gb, "GB:", [q.get(timeout=300) for _ in ps], flush=True)
        [p.join() for p in ps]
        os.unlink(path)
        if os.path.exists(path + ".pinned"): os.unlink(path + ".pinned")
