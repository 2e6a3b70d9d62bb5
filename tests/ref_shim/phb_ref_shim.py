"""pytest plugin (-p phb_ref_shim): installs paper_2404_18497_b200.compat_kernels
as ``pilothash._kernels`` before the reference package is imported, so the
reference's own test suite runs its construction / query path on the
B200 kernels. Counts the calls that reach the shim and
prints them at the end of the session. Test infrastructure only."""

import functools
import sys

from paper_2404_18497_b200 import _native, compat_kernels

_native.require_device()
_native.load()
CALLS = {"murmur3_many": 0, "build_partition_range": 0, "query_many_kernel": 0}


def _counted(name):
    fn = getattr(compat_kernels, name)

    @functools.wraps(fn)
    def w(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)

    return w


for _n in CALLS:
    setattr(compat_kernels, _n, _counted(_n))
sys.modules["pilothash._kernels"] = compat_kernels
print(f"phb_ref_shim: pilothash._kernels -> {compat_kernels.__file__} ({_native.LIB_PATH})",
      file=sys.stderr, flush=True)


def pytest_sessionfinish(session, exitstatus):
    import pilothash._kernels as k

    assert k is compat_kernels
    print("phb_ref_shim calls: " + " ".join(f"{a}={b}" for a, b in CALLS.items())
          + f" launches={_native.launch_count()}", file=sys.stderr, flush=True)
