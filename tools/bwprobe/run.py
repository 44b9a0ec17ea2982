import ctypes, os
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbwprobe.so"))
L.bw_probe.argtypes = [ctypes.c_size_t, ctypes.c_int]
L.bw_probe(1 << 31, 5)
