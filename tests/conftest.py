import os
import sys

# Simulated multi-rank tests (LocalTransport(fused=True)) run one CUDA stream
# per rank whose kernels wait on each other in-kernel; with the default 8
# hardware queues, more streams alias onto shared queues and a waiting
# kernel can block a peer's kernel queued behind it.  Must be set before CUDA
# initialises (importing torch does not initialise it).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and with CUDA 12 lazy module loading, the first launch of a kernel
# loads its module, which waits for the kernels already running on the
# device -- among them a simulated rank spinning on a barrier for a peer whose
# launch is now queued behind the load (NVIDIA's documented lazy-loading
# hazard for kernels that wait on each other).  Load eagerly.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")
