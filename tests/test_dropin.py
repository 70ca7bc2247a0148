"""The C++ drop-in (integration/cwgpu_process_query.cpp) inside the reference's own types:
cwgpu::process_query vs cwpir::process_query on a PirDatabase::setup database built by the
reference (byte payloads, perfect_map codewords), then the reference's extract().  Each case
answers two different databases that live in the same variable (same address, same parameters),
so a device copy keyed on the address would be caught, and runs on every visible GPU or on
several contexts of one GPU (the multi-device path, cwg_create_multi with device_ids = {0, 0})."""
import ctypes
import os

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

DROPIN = os.path.join(ROOT, "oracle", "_ref", "libcwgpu_dropin.so")


@pytest.mark.parametrize("n_dev", [0, 2], ids=["visible-gpus", "two-contexts-one-gpu"])
@pytest.mark.parametrize("N,L,bits,t,n,k,payload,target", [
    (2048, 3, 54, 12289, 30, 2, 16, 7),      # the reference's "BFV index pipeline" case (test_pir.cpp:311-330)
    (4096, 3, 36, 65537, 200, 2, 9000, 123),  # config-1 parameters, 2 plaintexts per row
])
def test_dropin_process_query_matches_reference(gpu, N, L, bits, t, n, k, payload, target, n_dev):
    if not os.path.exists(DROPIN):
        pytest.fail("drop-in harness not built (oracle/build_ref.sh after the product build)")
    lib = ctypes.CDLL(DROPIN)
    lib.dropin_last_error.restype = ctypes.c_char_p
    eq, ex = ctypes.c_int(), ctypes.c_int()
    rc = lib.dropin_check(ctypes.c_uint64(5), ctypes.c_uint32(N), ctypes.c_uint64(t), ctypes.c_uint32(L),
                          ctypes.c_uint32(bits), ctypes.c_uint64(n), ctypes.c_uint32(k), ctypes.c_uint32(payload),
                          ctypes.c_uint64(target), ctypes.c_int(n_dev), ctypes.byref(eq), ctypes.byref(ex))
    assert rc == 0, lib.dropin_last_error().decode()
    assert eq.value == 1, "cwgpu::process_query differs from cwpir::process_query"
    assert ex.value == 1, "extract() did not recover the row's payload"
