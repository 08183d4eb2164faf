"""Which NVML NVLink counters does this driver expose? (diagnostic for bench.nvlink_bytes)"""
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
names = [n for n in dir(pynvml) if n.startswith("NVML_FI_DEV_NVLINK")]
for n in sorted(names):
    fid = getattr(pynvml, n)
    for scope in (0, 0xFFFFFFFF):
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            if v.nvmlReturn == 0:
                print(n, fid, "scope", hex(scope), "ok", v.value.ullVal)
        except Exception as e:  # noqa: BLE001
            print(n, fid, "scope", hex(scope), "error", e)
for link in range(18):
    try:
        print("link", link, "state", pynvml.nvmlDeviceGetNvLinkState(h, link))
    except Exception as e:  # noqa: BLE001
        print("link", link, "state error", e)
        break
