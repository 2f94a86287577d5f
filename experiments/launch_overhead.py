import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblaunch_overhead.so"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
f = ctypes.c_float()
for coop in (0, 1):
    for threads, smem in ((288, 0), (288, 200 * 1024), (544, 200 * 1024)):
        for b2b in (1, 4):
            for fl in (0, 1):
                lib.run_empty(coop, threads, smem, 20, b2b, ctypes.byref(f), ctypes.c_void_p(flush.data_ptr() if fl else 0), ctypes.c_size_t(256 << 20))
                print(f"coop={coop} threads={threads} smem={smem//1024}KB launches={b2b} flush={fl}: {f.value*1e3:.1f} us")
