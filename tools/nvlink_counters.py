"""NVLink data-byte counters of one GPU through NVML (hardware counters, not
a profiler): cumulative bytes transmitted / received over all of the GPU's
NVLinks.  The bench reads them around its timed region at N>1 so the
sharded step's link traffic is measured, not inferred.

    python tools/nvlink_counters.py [--index 0]     # prints the current totals
"""
import json
import sys

try:
    import pynvml
except Exception:  # pragma: no cover - nvidia_ml_py is in the image
    pynvml = None

MAX_LINKS = 18


class NvLinkCounters:
    def __init__(self, index):
        self.ok = False
        self.error = None
        if pynvml is None:
            self.error = "pynvml missing"
            return
        try:
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.links = []
            for link in range(MAX_LINKS):
                try:
                    if pynvml.nvmlDeviceGetNvLinkState(self.h, link) == pynvml.NVML_FEATURE_ENABLED:
                        self.links.append(link)
                except pynvml.NVMLError:
                    break
            self.ok = bool(self.links)
            if not self.ok:
                self.error = "no active NVLink"
        except Exception as e:
            self.error = repr(e)[:200]

    def read(self):
        """(tx_bytes, rx_bytes) summed over the active links, or None."""
        if not self.ok:
            return None
        req = []
        for link in self.links:
            req.append((pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link))
            req.append((pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link))
        try:
            vals = pynvml.nvmlDeviceGetFieldValues(self.h, req)
        except Exception as e:
            self.error = repr(e)[:200]
            self.ok = False
            return None
        tx = rx = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            x = int(v.value.ullVal)
            if i % 2 == 0:
                tx += x
            else:
                rx += x
        # the THROUGHPUT_DATA counters are in KiB
        return tx * 1024, rx * 1024


def main():
    idx = int(sys.argv[sys.argv.index("--index") + 1]) if "--index" in sys.argv else 0
    c = NvLinkCounters(idx)
    print(json.dumps({"links": getattr(c, "links", []), "read": c.read(), "error": c.error}))


if __name__ == "__main__":
    main()
