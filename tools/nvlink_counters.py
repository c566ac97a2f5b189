"""NVLink data counters through NVML (measurement evidence for the NVLink roofline).

On the round-1 B200 boxes (driver 580) NVML answers NOT_SUPPORTED for these
fields and GPM sampling fails, so bench.py reports traffic = null for
multi-GPU runs; the helper stays so the field fills in where supported.

nvlink_bytes(dev) -> (tx_bytes, rx_bytes) cumulative NVLink *data* bytes of GPU
`dev`, summed over its links (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB
counters). bench.py reads them around the timed region to report the measured
link traffic per launch next to the algorithmic 2(P-1)/P S. Returns None when
NVML or the fields are unavailable.
"""
from __future__ import annotations

_h = {}


def _handle(dev: int):
    import pynvml
    if not _h:
        pynvml.nvmlInit()
    if dev not in _h:
        _h[dev] = pynvml.nvmlDeviceGetHandleByIndex(dev)
    return _h[dev]


def nvlink_bytes(dev: int, max_links: int = 18):
    try:
        import pynvml
        h = _handle(dev)
        tx = rx = 0
        ok = False
        for fid, acc in ((pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, "tx"),
                         (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, "rx")):
            reqs = []
            for link in range(max_links):
                reqs.append((fid, link))
            vals = pynvml.nvmlDeviceGetFieldValues(h, reqs)
            tot = 0
            for v in vals:
                if v.nvmlReturn != 0:
                    continue
                ok = True
                tot += int(v.value.ullVal)
            if acc == "tx":
                tx = tot
            else:
                rx = tot
        if not ok:
            return None
        return tx * 1024, rx * 1024
    except Exception:
        return None


if __name__ == "__main__":
    import sys
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    print(nvlink_bytes(d))

