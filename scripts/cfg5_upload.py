"""Config 5 index upload breakdown: host narrowing (int64 -> int16/int32
into pinned memory), PCIe copy, and the per-n-plet kernel, each alone."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_03381_b200 import _build, workloads  # noqa: E402


def main():
    _build.build()
    idx = np.ascontiguousarray(workloads.cfg5_nplets())
    src = torch.from_numpy(idx)
    res = {"threads": torch.get_num_threads()}
    for dt in (torch.int16, torch.int32):
        pin = torch.empty(src.shape, dtype=dt, pin_memory=True)
        dev = torch.empty(src.shape, dtype=dt, device="cuda")
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            pin.copy_(src)
            ts.append(time.perf_counter() - t0)
        res[f"narrow_{dt}_ms"] = min(ts) * 1e3
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.copy_(pin, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        res[f"h2d_{dt}_ms"] = min(ts) * 1e3
        res[f"h2d_{dt}_GBs"] = pin.numel() * pin.element_size() / min(ts) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
