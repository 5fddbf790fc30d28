"""Thread count of the oracle's library primitives (test infrastructure only): scipy.fft
runs with workers = every core this process may use (the CPU baseline uses all
affinity cores).  Library choice only -- no arithmetic of the method lives here."""

import os

WORKERS = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
