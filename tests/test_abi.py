"""CPU-only checks of the C ABI: the library builds for sm_100a, loads, exports
every symbol include/lamps.h declares, its struct layouts match the binding,
and host-side config validation works without a GPU (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "lamps.h")


@pytest.fixture(scope="module")
def L():
    from paper_2410_18248_b200 import lamps
    return lamps


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(lamps_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_the_five_calls():
    fns = declared_functions()
    for f in ("lamps_init", "lamps_submit", "lamps_api_return", "lamps_schedule_step", "lamps_free"):
        assert f in fns


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    out = subprocess.check_output(["nm", "-D", "--defined-only", L._build.LIB], text=True)
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    for f in declared_functions():
        assert f in exported, f
        assert getattr(lib, f)


def test_library_is_sm100a(L):
    L.lib()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L._build.LIB], text=True)
    assert "sm_100a" in out


def test_struct_layouts_match_header(L, tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "lamps.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(lamps_segment), sizeof(lamps_event),'
                   'sizeof(lamps_config), sizeof(lamps_step_out), sizeof(lamps_pool_io),'
                   'offsetof(lamps_config, stream));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)], text=True).split()]
    assert sizes == [ctypes.sizeof(L.lamps_segment), ctypes.sizeof(L.lamps_event),
                     ctypes.sizeof(L.lamps_config), ctypes.sizeof(L.lamps_step_out),
                     ctypes.sizeof(L.lamps_pool_io), L.lamps_config.stream.offset]
    assert L.SEGMENT_DTYPE.itemsize == sizes[0] and L.EVENT_DTYPE.itemsize == sizes[1]


def _cfg(L, **over):
    import gen
    d = gen.lib_config("C2")
    d.update(over)
    c = L.lamps_config()
    for k, v in d.items():
        setattr(c, k, v)
    return c


def test_workspace_query_needs_no_gpu(L):
    n = L.lamps_workspace_bytes(_cfg(L))
    assert n > 2048 * 7 * 4 and n % 256 == 0
    big = L.lamps_workspace_bytes(_cfg(L, capacity=1 << 20, id_bits=20, score_bits=35))
    assert big > 40 * (1 << 20)


@pytest.mark.parametrize("bad", [
    dict(capacity=3), dict(capacity=1 << 24), dict(block_tokens=12), dict(starvation_threshold=0),
    dict(max_batch=0), dict(max_batch=20000), dict(score_bits=40, id_bits=24), dict(id_bits=10),
    dict(A1=1 << 48), dict(SH=64), dict(c_other=1 << 32), dict(ticks_per_second=0.0),
    dict(ticks_per_second=float("inf")),
])
def test_config_validation(L, bad):
    c = _cfg(L, **bad)
    n = ctypes.c_size_t(0)
    assert L.lib().lamps_init(ctypes.byref(c), None, ctypes.byref(n), None) == L.LAMPS_EINVAL


def test_null_arguments(L):
    lib = L.lib()
    assert lib.lamps_init(None, None, None, None) == L.LAMPS_EINVAL
    assert lib.lamps_submit(None, None, 0, None) == L.LAMPS_EINVAL
    assert lib.lamps_schedule_step(None, None, 0, 0, None) == L.LAMPS_EINVAL
    assert lib.lamps_free(None) == L.LAMPS_EINVAL
    assert lib.lamps_last_error(None) == b"null handle"
    assert lib.lamps_version() >> 16 == 1


def test_no_cpu_fallback_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.LampsError):
        L.Scheduler(dict(capacity=16, max_batch=4, id_bits=23, score_bits=40))


def test_multi_shard_config_limits(L):
    """The P2P in-kernel merge stages world x K records on chip (<= 8192); the NCCL and
    loopback transports merge any exchange (the grid-wide merge by rank); local_ranks <= world."""
    nid = ctypes.create_string_buffer(128)
    n = ctypes.c_size_t(0)
    big_p2p = _cfg(L, max_batch=8192, world=8, rank=0, transport=L.LAMPS_XPORT_P2P)
    assert L.lib().lamps_init(ctypes.byref(big_p2p), None, ctypes.byref(n), None) == L.LAMPS_EINVAL
    big_nccl = _cfg(L, max_batch=8192, world=8, rank=0, transport=L.LAMPS_XPORT_NCCL)
    big_nccl.nccl_id = ctypes.cast(nid, ctypes.c_void_p)
    assert L.lib().lamps_init(ctypes.byref(big_nccl), None, ctypes.byref(n), None) == L.LAMPS_OK
    small = L.lamps_workspace_bytes(_cfg(L, max_batch=256, world=8, rank=0, transport=L.LAMPS_XPORT_LOOPBACK))
    large = L.lamps_workspace_bytes(_cfg(L, max_batch=8192, world=8, rank=0, transport=L.LAMPS_XPORT_LOOPBACK))
    assert large > small + 8 * 8 * 8192 * 4  # the merge-by-rank count matrix
    over = _cfg(L, world=4, rank=0, transport=L.LAMPS_XPORT_P2P, local_ranks=5)
    assert L.lib().lamps_init(ctypes.byref(over), None, ctypes.byref(n), None) == L.LAMPS_EINVAL
    ok = _cfg(L, world=8, rank=3, transport=L.LAMPS_XPORT_P2P, local_ranks=4, flags=L.LAMPS_SHARE_DEVICE)
    assert L.lib().lamps_init(ctypes.byref(ok), None, ctypes.byref(n), None) == L.LAMPS_OK


def test_large_pool_workspace(L):
    """Pools above the fused kernel's capacity carry the large-pool path's range regions."""
    n21 = L.lamps_workspace_bytes(_cfg(L, capacity=1 << 21, id_bits=21, score_bits=35))
    n20 = L.lamps_workspace_bytes(_cfg(L, capacity=1 << 20, id_bits=20, score_bits=35))
    assert n21 > 2 * n20
    forced = L.lamps_workspace_bytes(_cfg(L, flags=L.LAMPS_BIG_STEP))
    plain = L.lamps_workspace_bytes(_cfg(L, flags=L.LAMPS_MULTI_KERNEL))  # the 3-kernel path alone
    assert forced > plain + 148 * 10240 * 8  # V >= 148 range regions of 10240 keys


def test_group_step_async_rejects_bad_groups(L):
    """lamps_group_step_async validates before touching any handle (NULL / empty groups)."""
    kv = (ctypes.c_uint64 * 1)(0)
    assert L.lib().lamps_group_step_async(None, 1, kv) == L.LAMPS_EINVAL
    hs = (ctypes.c_void_p * 1)(None)
    assert L.lib().lamps_group_step_async(hs, 1, kv) == L.LAMPS_EINVAL
    assert L.lib().lamps_group_step_async(hs, 0, kv) == L.LAMPS_EINVAL
