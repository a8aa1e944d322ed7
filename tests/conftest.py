import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libstgmg.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    # OpenBLAS with every logical CPU is pathologically slow for the oracle's LAPACK calls on shared hosts (measured
    # here: a 1000^2 inverse 0.09 s on 4 threads, 1.4 s on 8); half the CPUs keeps the CPU suite within minutes.
    try:
        from threadpoolctl import threadpool_limits
        session.config._stgmg_blas_limit = threadpool_limits(max(1, (os.cpu_count() or 2) // 2))
    except Exception:
        pass
