"""ctypes binding of the sm_100a C-ABI library (include/bddc_b200.h).

The signatures are parsed from the header, so the header is the single
source of truth for the boundary.  Loading fails loudly: there is no CPU
fallback anywhere in the package.
"""

import ctypes
import os
import re

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BDDC_LIB") or os.path.join(HERE, "_bddc_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "bddc_b200.h")

_CTYPES = {
    "int": ctypes.c_int,
    "long long": ctypes.c_longlong,
    "double": ctypes.c_double,
    "cudaStream_t": ctypes.c_void_p,
}


def parse_header(path=HEADER):
    """{name: (restype, [argtypes])} for every bddc_* function declared."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"(int|long long)\s+(bddc_\w+)\s*\(([^)]*)\)\s*;", text):
        ret, name, args = m.group(1), m.group(2), m.group(3)
        types = []
        if args.strip() in ("", "void"):
            out[name] = (_CTYPES[ret], types)
            continue
        for a in args.split(","):
            a = " ".join(a.replace("const", " ").split())
            if "*" in a:
                types.append(ctypes.c_void_p)
            else:
                base = a.rsplit(" ", 1)[0]
                types.append(_CTYPES[base])
        out[name] = (_CTYPES[ret], types)
    return out


class _Lib:
    def __init__(self):
        self._dll = None
        self._sigs = None

    def load(self):
        if self._dll is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA extension {LIB_PATH} is missing: build it with "
                    "`python -m paper_2501_01676_b200.build` (there is no CPU fallback)")
            dll = ctypes.CDLL(LIB_PATH)
            sigs = parse_header()
            for name, (ret, args) in sigs.items():
                fn = getattr(dll, name)
                fn.restype = ret
                fn.argtypes = args
            self._dll, self._sigs = dll, sigs
        return self._dll

    def __getattr__(self, name):
        if not name.startswith("bddc_"):
            raise AttributeError(name)
        dll = self.load()
        fn = getattr(dll, name)
        return _checked(name, fn)


def _conv(a):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            raise ValueError("device tensor expected")
        return ctypes.c_void_p(a.data_ptr())
    return a


# Optional per-entry-point GPU time profile (tools/kernel_profile.py): CUDA
# events around every C-ABI call on the current stream, summed by name.
_PROFILE = {"on": False, "events": []}


def profile(enable=True):
    _PROFILE["on"] = bool(enable)
    _PROFILE["events"] = []


def profile_report():
    """{name: (calls, ms)} of the calls recorded since profile(True)."""
    out = {}
    evs = _PROFILE["events"]
    if evs:
        evs[-1][2].synchronize()
    for name, e0, e1 in evs:
        c, t = out.get(name, (0, 0.0))
        out[name] = (c + 1, t + e0.elapsed_time(e1))
    return out


def _checked(name, fn):
    def call(*args):
        if _PROFILE["on"] and not name.startswith(("bddc_ws_", "bddc_launch")):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn(*[_conv(a) for a in args])
            e1.record()
            _PROFILE["events"].append((name, e0, e1))
        else:
            rc = fn(*[_conv(a) for a in args])
        if isinstance(rc, int) and not name.startswith(("bddc_ws_", "bddc_launch")) and rc < 0:
            raise RuntimeError(f"{name}: CUDA launch failed ({torch.cuda.get_device_name()} "
                               f"error {-rc})")
        return rc
    return call


lib = _Lib()


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_01676_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    lib.load()
