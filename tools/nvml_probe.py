"""Which NVML NVLink byte counters this GPU/driver exposes (field id, scope) and their values."""
import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
print("driver", nv.nvmlSystemGetDriverVersion())
for name in ("NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES",
             "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
             "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX",
             "NVML_FI_DEV_NVLINK_LINK_COUNT"):
    fid = getattr(nv, name, None)
    if fid is None:
        print(name, "not in pynvml")
        continue
    for scope in (0xFFFFFFFF, 0, 1, 17):
        v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
        print(name, fid, hex(scope), "ret", v.nvmlReturn, "type", v.valueType, "ull", v.value.ullVal)
try:
    for link in range(2):
        print("link", link, "state", nv.nvmlDeviceGetNvLinkState(h, link))
except Exception as e:
    print("nvlink state", e)
