import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_sessionfinish(session, exitstatus):
    """Write the parity maxima the GPU tests recorded (tests/_harness.RECORD) to $TBA_PARITY_OUT."""
    out = os.environ.get("TBA_PARITY_OUT")
    if not out:
        return
    try:
        from tests import _harness as H
    except Exception:  # pragma: no cover
        return
    if not H.RECORD:
        return
    import json
    import platform
    meta = dict(cores=H.n_workers(), host=platform.processor() or platform.machine(), exitstatus=int(exitstatus))
    try:
        import torch
        if torch.cuda.is_available():
            meta["gpu"] = torch.cuda.get_device_name(0)
    except Exception:  # pragma: no cover
        pass
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with open(out, "w") as f:
        json.dump(dict(meta=meta, records=H.RECORD), f, indent=1)
