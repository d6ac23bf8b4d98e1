"""Probe: write-only HBM bandwidth (the roofline of an output-only kernel).

torch fill_ (a plain store kernel) and a 256-bit-store kernel of our own
(st.global.v8.b32, the instruction the generator flushes with), 32 GiB, best
of 5 by CUDA events."""
import json
import os
import subprocess
import sys
import tempfile

import torch

SRC = r'''
#include <stdint.h>
extern "C" __global__ void fill256(uint32_t* p, uint64_t n32) {
  uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
  for (; i + 8 <= n32; i += stride) {
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + i), "r"((uint32_t)i));
  }
}
'''


def main():
    dev = torch.device("cuda", 0)
    n = 32 << 30
    buf = torch.empty(n, dtype=torch.uint8, device=dev)
    res = {}

    def best(fn, reps=5):
        fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        return min(ts)

    res["torch_fill_gbs"] = n / best(lambda: buf.fill_(7)) / 1e9
    with tempfile.TemporaryDirectory() as d:
        cu, cubin = os.path.join(d, "f.cu"), os.path.join(d, "f.cubin")
        open(cu, "w").write(SRC)
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-o",
                        cubin, cu], check=True)
        from cuda.bindings import driver as cu_drv
        cu_drv.cuInit(0)
        err, mod = cu_drv.cuModuleLoad(cubin.encode())
        err, fn = cu_drv.cuModuleGetFunction(mod, b"fill256")
        import ctypes
        ptr = ctypes.c_uint64(buf.data_ptr())
        n32 = ctypes.c_uint64(n // 4)
        args = (ctypes.c_void_p * 2)(ctypes.addressof(ptr), ctypes.addressof(n32))
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        stream = torch.cuda.current_stream(dev).cuda_stream

        def launch():
            cu_drv.cuLaunchKernel(fn, sms * 8, 1, 1, 256, 1, 1, 0, stream, ctypes.addressof(args), 0)
        res["st256_fill_gbs"] = n / best(launch) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
