import pynvml as n
n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(0)
for f in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX"):
    fid = getattr(n, f)
    for scope in (0, 1, 0xFFFFFFFF):
        v = n.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
        print(f, scope, v.nvmlReturn, v.valueType, v.value.ullVal)
try:
    print("links active:", sum(1 for l in range(18) if n.nvmlDeviceGetNvLinkState(h, l) == 1))
except Exception as e:
    print("state err", e)
