import time, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
for f in (lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)):
    t=time.perf_counter()
    for _ in range(10): f()
    print((time.perf_counter()-t)/10*1e3, "ms per call")
