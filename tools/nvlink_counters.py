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
        ok = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            ok += 1
            x = int(v.value.ullVal)
            if i % 2 == 0:
                tx += x
            else:
                rx += x
        if ok == 0:
            self.error = f"NVML returned no NVLink throughput fields (codes {[v.nvmlReturn for v in vals][:4]})"
            self.ok = False
            return None
        # the THROUGHPUT_DATA counters are in KiB
        return tx * 1024, rx * 1024


def main():
    idx = int(sys.argv[sys.argv.index("--index") + 1]) if "--index" in sys.argv else 0
    c = NvLinkCounters(idx)
    out = {"links": getattr(c, "links", []), "read": c.read(), "error": c.error}
    if c.ok or getattr(c, "links", None):
        raw = {}
        for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX",
                     "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES"):
            fid = getattr(pynvml, name, None)
            if fid is None:
                continue
            for scope in (0, 0xFFFFFFFF):
                try:
                    v = pynvml.nvmlDeviceGetFieldValues(c.h, [(fid, scope)])[0]
                    raw[f"{name}@{scope}"] = (v.nvmlReturn, int(v.value.ullVal))
                except Exception as e:
                    raw[f"{name}@{scope}"] = repr(e)[:80]
        out["raw"] = raw
    print(json.dumps(out))


if __name__ == "__main__":
    main()
