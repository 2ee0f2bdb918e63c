"""K6 CRC-32 throughput (CUDA events around actc_crc32's launch, inputs in
HBM, > L2) against zlib.crc32 on the host, and to_bytes of a device-resident
stream (device CRC + one D2H copy) against the host-CRC serialisation."""
import json
import os
import sys
import time
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib, codec as pc  # noqa: E402

res = {}
for mb in (64, 1024):
    n = mb << 20
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        pc.crc32_device(t, n)
    _lib.timing_enable(True)
    _lib.kernel_stats()
    K = 10
    for _ in range(K):
        pc.crc32_device(t, n)
    st = _lib.kernel_stats()
    _lib.timing_enable(False)
    ms = st["crc"][1] / st["crc"][0]
    host = t[: min(n, 256 << 20)].cpu().numpy().tobytes()
    h0 = time.perf_counter()
    zlib.crc32(host)
    hz = time.perf_counter() - h0
    res[f"{mb}MB"] = {"device_ms": ms, "device_GBps": n / ms / 1e6, "zlib_GBps": len(host) / hz / 1e9}
# to_bytes of a conv-sized stream
x = torch.randn(256, 64, 55, 55, device="cuda").relu_()
c, rep = pb.compress(x, pb.CodecParams(eb=1e-3))
c.to_bytes()
h0 = time.perf_counter()
blob = c.to_bytes()
t_dev = time.perf_counter() - h0
h0 = time.perf_counter()
zlib.crc32(blob[:-4])
t_z = time.perf_counter() - h0
res["to_bytes"] = {"blob_MB": len(blob) / 1e6, "to_bytes_s": t_dev, "host_zlib_crc_alone_s": t_z}
print(json.dumps(res))
