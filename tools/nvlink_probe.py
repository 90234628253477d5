"""Which NVML NVLink byte counters move on this pool's B200s, and by how much.

One process, two GPUs: a known number of bytes is copied GPU0 -> GPU1 (peer
copy over NVLink); the NVML field values of every link are read before and
after on both GPUs and the deltas printed next to the copied bytes.  bench.py
uses the field that reports the copy faithfully to count the NVLink bytes of
the multi-GPU exchange in its timed region.
"""
import json
import sys

import pynvml as nv
import torch

FIELDS = {
    "THROUGHPUT_DATA_TX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
    "THROUGHPUT_DATA_RX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
    "THROUGHPUT_RAW_TX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX,
    "THROUGHPUT_RAW_RX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX,
    "COUNT_XMIT_BYTES": nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
    "COUNT_RCV_BYTES": nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
}
NLINK = 18
ERRS = {}


def read(h):
    out = {}
    for name, fid in FIELDS.items():
        vals = []
        for link in list(range(NLINK)) + [0xFFFFFFFF]:
            try:
                fv = nv.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                if fv.nvmlReturn != 0:
                    vals.append(None)
                    ERRS.setdefault(name, set()).add(int(fv.nvmlReturn))
                    continue
                vt = fv.valueType
                v = {0: fv.value.dVal, 1: fv.value.uiVal, 2: fv.value.ulVal, 3: fv.value.ullVal,
                     4: fv.value.sllVal}.get(vt, fv.value.ullVal)
                vals.append(int(v))
            except Exception as e:  # noqa: BLE001
                vals.append(None)
        out[name] = vals
    return out


def smi():
    import subprocess
    r = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True)
    r1 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "1"], capture_output=True, text=True)
    return r.stdout + r.stderr, r1.stdout + r1.stderr


def delta(a, b):
    return {k: [(y - x) if (x is not None and y is not None) else None for x, y in zip(a[k], b[k])] for k in a}


def main():
    nv.nvmlInit()
    n = torch.cuda.device_count()
    hs = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(n)]
    nbytes = int(float(sys.argv[1]) if len(sys.argv) > 1 else 4e9)
    src = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda:0").fill_(1.0)
    dst = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda:1")
    dst.copy_(src)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    before = [read(h) for h in hs[:2]]
    smi0 = smi()
    reps = 5
    for _ in range(reps):
        dst.copy_(src)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    after = [read(h) for h in hs[:2]]
    smi1 = smi()
    res = {"copied_bytes": nbytes * reps, "direction": "gpu0 -> gpu1",
           "delta_gpu0": delta(before[0], after[0]), "delta_gpu1": delta(before[1], after[1])}
    for g in ("delta_gpu0", "delta_gpu1"):
        res[g + "_sum_links"] = {k: sum(x for x in v[:NLINK] if x is not None) for k, v in res[g].items()}
    res["nvml_errors"] = {k: sorted(v) for k, v in ERRS.items()}
    st = []
    for link in range(NLINK):
        try:
            st.append(int(nv.nvmlDeviceGetNvLinkState(hs[0], link)))
        except Exception as e:  # noqa: BLE001
            st.append(str(e))
    res["nvlink_state_gpu0"] = st
    res["smi_before"], res["smi_after"] = smi0, smi1
    print(json.dumps(res))


if __name__ == "__main__":
    main()
