"""Where the e2e time goes beyond the device time: python wall (ctypes call) vs the C wall clock
(fsw_invoke entry -> output in the caller buffer, stats.total_ms) vs the CUDA-event device time."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2306_03622_b200 import Runtime

with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    for name in sys.argv[1:] or ["mlp", "bert-base"]:
        spec = synth.build_model(name)
        mid = rt.register_spec(spec, spec.build_weights(), link_code=True)
        x = spec.make_input()
        info = rt.model_info(mid)
        out = np.empty(info["output_bytes"] // 4, np.float32)
        for cold in (False, True):
            py, c, dev, hs, hw = [], [], [], [], []
            for i in range(40):
                if cold:
                    rt.evict(mid)
                t0 = time.perf_counter()
                st = rt.invoke_plain(mid, x, out)
                py.append((time.perf_counter() - t0) * 1e3)
                c.append(st["total_ms"]); dev.append(st["device_ms"]); hs.append(st["host_setup_ms"]); hw.append(st["host_wait_ms"])
            m = lambda a: round(float(np.median(a[5:])), 4)
            print(name, "cold" if cold else "warm", "python", m(py), "C total", m(c), "device", m(dev),
                  "host setup", m(hs), "host wait", m(hw), flush=True)
        rt.unregister(mid)
