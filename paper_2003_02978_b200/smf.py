"""Thin Python binding of libsmf.so (include/smf.h) -- argument marshalling only.

Every step of the retrieval runs in the library's CUDA kernels; torch is used
for device memory and streams. There is no CPU fallback: importing this module
fails loudly when libsmf.so is missing, and calls fail when no CUDA device is
present.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsmf.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsmf.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i = ctypes.c_int
_d = ctypes.c_double

SYMBOLS = {
    # name: (restype, argtypes)
    "smf_create": (_i, [ctypes.POINTER(_vp), _i]),
    "smf_destroy": (None, [_vp]),
    "smf_set_absorption": (_i, [_vp, _vp, _i]),
    "smf_set_regularisation": (_i, [_vp, _d, _d, _d]),
    "smf_set_iterations": (_i, [_vp, _i, _i, _i]),
    "smf_workspace_bytes": (_i, [_vp, _i, _i, ctypes.POINTER(ctypes.c_size_t)]),
    "smf_supported_bands": (_i, [_i]),
    "smf_retrieve": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "smf_synchronize": (_i, [_vp, _vp, _vp, _i, ctypes.POINTER(_i)]),
    "smf_retrieve_host": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp]),
    "smf_column_model": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp]),
    "smf_initial_statistics": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp]),
    "smf_last_launch_count": (_i, [_vp]),
    "smf_set_stats_kernel": (_i, [_vp, _i]),
    "smf_set_energy_trace": (_i, [_vp, _i]),
    "smf_set_grouping": (_i, [_vp, _i]),
    "smf_set_nodata": (_i, [_vp, _i, ctypes.c_float]),
    "smf_convert_layout": (_i, [_vp, _i, _i, _i, _i, _vp, _vp]),
    "smf_group_partitions": (_i, [_i, _i, ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "smf_energy_trace": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "smf_stats_kernel_used": (_i, [_vp]),
    "smf_host_chunk_cols": (_i, [_vp, _i, ctypes.POINTER(_i)]),
    "smf_set_graph": (_i, [_vp, _i]),
    "smf_set_covariance_check": (_i, [_vp, _i]),
    "smf_set_diagnostics": (_i, [_vp, _i]),
    "smf_set_nvtx": (_i, [_vp, _i]),
    "smf_iteration_diagnostics": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "smf_profile_enable": (_i, [_vp, _i]),
    "smf_profile_read": (_i, [_vp, _i, ctypes.POINTER(_d), ctypes.POINTER(_i)]),
    "smf_status_string": (ctypes.c_char_p, [_i]),
    "smf_last_error": (ctypes.c_char_p, [_vp]),
    "smf_abi_version": (_i, []),
}
for _name, (_res, _args) in SYMBOLS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

SMF_OK, SMF_ERR_INVALID_ARGUMENT, SMF_ERR_NOT_CONFIGURED, SMF_ERR_SHAPE, SMF_ERR_NUMERICAL, SMF_ERR_CUDA, \
    SMF_ERR_OUT_OF_MEMORY = range(7)
COLUMN_STATUS = {0: "OK", 1: "NONFINITE", 2: "DEGENERATE_MEAN", 3: "NOT_SPD", 4: "DEGENERATE_TARGET",
                 5: "INSUFFICIENT"}


class SMFError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_lib.smf_status_string(code).decode()}: {msg}")
        self.code = code


def abi_version() -> int:
    return _lib.smf_abi_version()


def supported_bands(bands: int) -> bool:
    return bool(_lib.smf_supported_bands(int(bands)))


LAYOUTS = {"BIL": 0, "BIP": 1}


def convert_layout(cube, layout, out=None, stream=None):
    """Device cube as stored on disk -> retrieval layout [samples][lines][bands]:
    BIL [lines][bands][samples] or BIP [lines][samples][bands] (smf_convert_layout)."""
    import torch
    lines = cube.shape[0]
    samples, bands = (cube.shape[2], cube.shape[1]) if layout == "BIL" else (cube.shape[1], cube.shape[2])
    if out is None:
        out = torch.empty((samples, lines, bands), dtype=torch.float32, device=cube.device)
    st = stream if stream is not None else torch.cuda.current_stream(cube.device)
    rc = _lib.smf_convert_layout(_ptr(cube), lines, samples, bands, LAYOUTS[layout], _ptr(out),
                                 ctypes.c_void_p(st.cuda_stream))
    if rc != SMF_OK:
        raise SMFError(rc, "convert_layout")
    return out


def group_partitions(cols: int, group: int) -> list:
    """First column of every partition for detector grouping (smf_group_partitions)."""
    n = _i()
    if _lib.smf_group_partitions(int(cols), int(group), ctypes.byref(n), None) != SMF_OK:
        raise SMFError(SMF_ERR_INVALID_ARGUMENT, "bad grouping request")
    first = (_i * max(n.value, 1))()
    _lib.smf_group_partitions(int(cols), int(group), ctypes.byref(n), first)
    return list(first[: n.value])


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _record(tensors, stream, device):
    """Tensors allocated on torch's current stream but used by kernels on `stream`: tell
    the caching allocator, so their memory is not handed out again before `stream` is done."""
    import torch
    if stream != torch.cuda.current_stream(device):
        for t in tensors:
            t.record_stream(stream)


class Retriever:
    """A library context (smf_ctx) bound to the current CUDA device."""

    STATS_KERNELS = {"auto": 0, "ffma": 1, "tensor": 2, "int8": 3}
    COV_CHECKS = {"off": 0, "auto": 1, "always": 2}

    def __init__(self, bands, s, n_iter=30, use_sparsity=True, use_albedo=True, eps=1e-2, ridge_rel=0.0,
                 r_floor=0.05, stats_kernel="auto", energy=False, group=1, nodata=None, graph=False,
                 cov_check="auto", diagnostics=False, nvtx=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("smf needs a CUDA device (no CPU fallback)")
        self.bands = int(bands)
        h = _vp()
        self._check(_lib.smf_create(ctypes.byref(h), self.bands), None)
        self._h = h
        s = np.ascontiguousarray(s, dtype=np.float32)
        self._check(_lib.smf_set_absorption(self._h, s.ctypes.data_as(_vp), self.bands))
        self._check(_lib.smf_set_regularisation(self._h, float(eps), float(ridge_rel), float(r_floor)))
        self._check(_lib.smf_set_iterations(self._h, int(n_iter), int(bool(use_sparsity)), int(bool(use_albedo))))
        self._check(_lib.smf_set_stats_kernel(self._h, self.STATS_KERNELS[stats_kernel]))
        self._check(_lib.smf_set_energy_trace(self._h, int(bool(energy))))
        self._check(_lib.smf_set_grouping(self._h, int(group)))
        self._check(_lib.smf_set_nodata(self._h, int(nodata is not None),
                                        float(nodata) if nodata is not None else -9999.0))
        self._check(_lib.smf_set_graph(self._h, int(bool(graph))))
        self._check(_lib.smf_set_covariance_check(self._h, self.COV_CHECKS[cov_check]))
        self._check(_lib.smf_set_diagnostics(self._h, int(bool(diagnostics))))
        if nvtx is not None:
            self._check(_lib.smf_set_nvtx(self._h, int(bool(nvtx))))
        self.group = int(group)
        self.n_iter = int(n_iter)

    def energy_trace(self, workspace, cols, pixels, stream=None):
        """Eq. 8 energy per iteration and partition (fp64 [n_iter + 1][partitions]; one
        partition per column unless grouped) of the last retrieve that used `workspace`
        (requires energy=True)."""
        import torch
        nparts = len(group_partitions(cols, self.group))
        out = torch.empty((self.n_iter + 1, nparts), dtype=torch.float64, device=workspace.device)
        st = stream if stream is not None else torch.cuda.current_stream(workspace.device)
        self._check(_lib.smf_energy_trace(self._h, _ptr(workspace), cols, pixels, _ptr(out),
                                          ctypes.c_void_p(st.cuda_stream)))
        return out

    def iteration_diagnostics(self, workspace, cols, pixels, stream=None):
        """Per-iteration records of the last retrieve that used `workspace` (requires
        diagnostics=True), each [n_iter + 1][partitions]: nonzero count of alpha^k (int64),
        q^k (fp64), partition status (int32), cumulative literal covariance checks (int32)."""
        import torch
        nparts = len(group_partitions(cols, self.group))
        dev = workspace.device
        shape = (self.n_iter + 1, nparts)
        out = {"nnz": torch.empty(shape, dtype=torch.int64, device=dev),
               "q": torch.empty(shape, dtype=torch.float64, device=dev),
               "status": torch.empty(shape, dtype=torch.int32, device=dev),
               "literal": torch.empty(shape, dtype=torch.int32, device=dev)}
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        self._check(_lib.smf_iteration_diagnostics(self._h, _ptr(workspace), cols, pixels, _ptr(out["nnz"]),
                                                   _ptr(out["q"]), _ptr(out["status"]), _ptr(out["literal"]),
                                                   ctypes.c_void_p(st.cuda_stream)))
        return out

    @property
    def stats_kernel_used(self) -> str:
        """'tensor' (tcgen05 kind::tf32, split), 'int8' (tcgen05 kind::i8, wide path) or 'ffma':
        the kernel computing mu0, C0."""
        return {1: "ffma", 2: "tensor", 3: "int8"}[_lib.smf_stats_kernel_used(self._h)]

    def _check(self, rc, h="self"):
        if rc != SMF_OK:
            msg = _lib.smf_last_error(self._h).decode() if h == "self" and getattr(self, "_h", None) else ""
            raise SMFError(rc, msg)

    def close(self):
        lib = globals().get("_lib")   # None during interpreter shutdown
        if getattr(self, "_h", None) and lib is not None:
            lib.smf_destroy(self._h)
        self._h = None

    __del__ = close

    @property
    def last_launch_count(self) -> int:
        return _lib.smf_last_launch_count(self._h)

    KERNELS = {"k1_stats": 0, "k2_init": 1, "k2_update": 2, "k3_sweep": 3}

    def profile_enable(self, on=True):
        self._check(_lib.smf_profile_enable(self._h, int(bool(on))))

    def profile_read(self):
        """{kernel: (total_ms, launches)} since the last profile_enable (synchronises)."""
        out = {}
        for name, kind in self.KERNELS.items():
            ms, n = _d(), _i()
            self._check(_lib.smf_profile_read(self._h, kind, ctypes.byref(ms), ctypes.byref(n)))
            out[name] = (ms.value, n.value)
        return out

    def workspace_bytes(self, cols, pixels) -> int:
        n = ctypes.c_size_t()
        self._check(_lib.smf_workspace_bytes(self._h, int(cols), int(pixels), ctypes.byref(n)))
        return n.value

    def alloc_workspace(self, cols, pixels, device=None):
        import torch
        return torch.empty(self.workspace_bytes(cols, pixels), dtype=torch.uint8,
                           device=device or torch.cuda.current_device())

    def retrieve(self, radiance, enhancement=None, albedo=None, workspace=None, status=None, stream=None):
        """radiance: CUDA fp32 tensor [cols][pixels][bands] (contiguous). Returns
        (enhancement, albedo, column_status) CUDA tensors; asynchronous on `stream`
        (default: torch's current stream)."""
        import torch
        assert radiance.is_cuda and radiance.dtype == torch.float32 and radiance.is_contiguous()
        cols, pixels, bands = radiance.shape
        if bands != self.bands:
            raise SMFError(SMF_ERR_SHAPE, f"bands {bands} != {self.bands}")
        dev = radiance.device
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        made = []   # allocated here on torch's current stream but used on `st`
        if enhancement is None:
            enhancement = torch.empty((cols, pixels), dtype=torch.float32, device=dev)
            made.append(enhancement)
        if albedo is None:
            albedo = torch.empty((cols, pixels), dtype=torch.float32, device=dev)
            made.append(albedo)
        if workspace is None:
            workspace = self.alloc_workspace(cols, pixels, dev)
            made.append(workspace)
        if status is None:
            status = torch.empty(cols, dtype=torch.int32, device=dev)
            made.append(status)
        _record(made, st, dev)
        self._check(_lib.smf_retrieve(self._h, _ptr(radiance), cols, pixels, _ptr(enhancement), _ptr(albedo),
                                      _ptr(workspace), _ptr(status), ctypes.c_void_p(st.cuda_stream)))
        return enhancement, albedo, status

    def synchronize(self, status, stream=None):
        """Wait for the stream; return the first failed column (-1 if none)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(status.device)
        first = ctypes.c_int(-1)
        rc = _lib.smf_synchronize(self._h, ctypes.c_void_p(st.cuda_stream), _ptr(status), status.numel(),
                                  ctypes.byref(first))
        if rc not in (SMF_OK, SMF_ERR_NUMERICAL):
            self._check(rc)
        return first.value

    def retrieve_host(self, radiance, enhancement=None, albedo=None, status=None):
        """Host (numpy) fp32 [cols][pixels][bands] in, host maps out; includes the
        host<->device copies. Returns (enhancement, albedo, column_status, rc)."""
        radiance = np.ascontiguousarray(radiance, dtype=np.float32)
        cols, pixels, bands = radiance.shape
        if enhancement is None:
            enhancement = np.empty((cols, pixels), np.float32)
        if albedo is None:
            albedo = np.empty((cols, pixels), np.float32)
        if status is None:
            status = np.empty(cols, np.int32)
        rc = _lib.smf_retrieve_host(self._h, radiance.ctypes.data_as(_vp), cols, pixels,
                                    enhancement.ctypes.data_as(_vp), albedo.ctypes.data_as(_vp),
                                    status.ctypes.data_as(_vp))
        if rc not in (SMF_OK, SMF_ERR_NUMERICAL):
            self._check(rc)
        return enhancement, albedo, status, rc

    def host_chunk_cols(self, cols: int) -> int:
        """Columns per chunk that retrieve_host streams for a cube of `cols` columns."""
        n = _i()
        self._check(_lib.smf_host_chunk_cols(self._h, int(cols), ctypes.byref(n)))
        return n.value

    def retrieve_host_ptr(self, rad_ptr, cols, pixels, enh_ptr, alb_ptr, status_ptr):
        """Same as retrieve_host on raw host pointers (e.g. pinned torch tensors)."""
        rc = _lib.smf_retrieve_host(self._h, ctypes.c_void_p(rad_ptr), int(cols), int(pixels),
                                    ctypes.c_void_p(enh_ptr), ctypes.c_void_p(alb_ptr), ctypes.c_void_p(status_ptr))
        if rc not in (SMF_OK, SMF_ERR_NUMERICAL):
            self._check(rc)
        return rc

    def initial_statistics(self, radiance, workspace=None, stream=None):
        """mu0 (fp64 [cols][bands]) and C0 (fp64 [cols][bands][bands]) from the K1 kernel."""
        import torch
        cols, pixels, bands = radiance.shape
        mean = torch.empty((cols, bands), dtype=torch.float64, device=radiance.device)
        cov = torch.empty((cols, bands, bands), dtype=torch.float64, device=radiance.device)
        st = stream if stream is not None else torch.cuda.current_stream(radiance.device)
        made = [mean, cov]
        if workspace is None:
            workspace = self.alloc_workspace(cols, pixels, radiance.device)
            made.append(workspace)
        _record(made, st, radiance.device)
        self._check(_lib.smf_initial_statistics(self._h, _ptr(radiance), cols, pixels, _ptr(mean), _ptr(cov),
                                                _ptr(workspace), ctypes.c_void_p(st.cuda_stream)))
        return mean, cov

    def column_model(self, workspace, cols, pixels, stream=None):
        """mu^{N_iter} (fp64 [partitions][bands]) and q^{N_iter} (fp64 [partitions]) of the last
        retrieve (one partition per column unless grouped)."""
        import torch
        nparts = len(group_partitions(cols, self.group))
        mu = torch.empty((nparts, self.bands), dtype=torch.float64, device=workspace.device)
        q = torch.empty(nparts, dtype=torch.float64, device=workspace.device)
        st = stream if stream is not None else torch.cuda.current_stream(workspace.device)
        self._check(_lib.smf_column_model(self._h, _ptr(workspace), cols, pixels, _ptr(mu), _ptr(q),
                                          ctypes.c_void_p(st.cuda_stream)))
        return mu, q


def retrieve(radiance, s, **kw):
    """One-shot convenience: build a context, run, synchronise."""
    r = Retriever(radiance.shape[2], s, **kw)
    enh, alb, st = r.retrieve(radiance)
    r.synchronize(st)
    return enh, alb, st
