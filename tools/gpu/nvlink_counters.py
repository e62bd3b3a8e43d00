"""NVLink data counters of every visible GPU (NVML field values), as JSON: per GPU the
sum over links of transmitted / received data bytes (COUNT_XMIT/RCV_BYTES) and the
THROUGHPUT_DATA_TX/RX counters (KiB), so a before/after pair around a run gives the
bytes that crossed NVLink."""
import json
import sys

import pynvml as N

pynvml_fields = [("xmit_bytes", N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES),
                 ("rcv_bytes", N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES),
                 ("data_tx_kib", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX),
                 ("data_rx_kib", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX)]
N.nvmlInit()
out = {}
for i in range(N.nvmlDeviceGetCount()):
    h = N.nvmlDeviceGetHandleByIndex(i)
    row = {}
    for name, fid in pynvml_fields:
        total, err = 0, None
        for link in range(18):
            try:
                v = N.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                if v.nvmlReturn == 0:
                    total += int(v.value.ullVal)
                else:
                    err = v.nvmlReturn
            except Exception as e:  # noqa: BLE001
                err = str(e)
        row[name] = total
        if err is not None and total == 0:
            row[name + "_err"] = str(err)
    out[i] = row
print(json.dumps(out))
