"""The C-ABI boundary on CPU: the library loads without a GPU, exports every
symbol include/kvx.h declares, and validates arguments before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2502_09334_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvx.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(kvx_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("kvx_quant_pack", "kvx_dequant_scatter_paged", "kvx_enable_peer",
                 "kvx_copy_peer", "kvx_ipc_get_handle", "kvx_ipc_open", "kvx_stream_signal",
                 "kvx_stream_wait", "kvx_strerror"):
        assert must in syms


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.SO_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (kvx_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_sm100a_cubin_embedded():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_strerror(lib):
    assert lib.kvx_version() >= 100
    assert _lib.strerror(0) == "ok"
    assert "invalid" in _lib.strerror(_lib.KVX_ERR_INVALID_ARG)
    assert "peer" in _lib.strerror(_lib.KVX_ERR_NO_PATH)


def test_packed_sizes(lib):
    c, s, z = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rows = 32 * 2 * 512 * 32  # cfg1 rows
    assert lib.kvx_packed_sizes(rows, 128, 128, 4, ctypes.byref(c), ctypes.byref(s), ctypes.byref(z)) == 0
    assert c.value == 67_108_864 and s.value == z.value == rows * 2
    assert c.value + s.value + z.value == 71_303_168  # SURVEY 8(d) cfg1 packed bytes
    assert lib.kvx_packed_sizes(rows, 128, 128, 16, ctypes.byref(c), ctypes.byref(s), ctypes.byref(z)) == 0
    assert c.value == 268_435_456 and s.value == 0


@pytest.mark.parametrize("bits,group,head_dim", [(5, 128, 128), (4, 96, 128), (4, 128, 64),
                                                 (4, 64, 100), (3, 32, 128)])
def test_invalid_format_rejected_before_cuda(lib, bits, group, head_dim):
    rc = lib.kvx_quant_pack(16, 16, 0, None, 1, 1, 1, head_dim, group, bits, 16, 16, 16, 0, 0, 0,
                            None)
    assert rc == _lib.KVX_ERR_INVALID_ARG
    rc = lib.kvx_dequant_scatter_paged(16, 16, 16, 0, None, 1, 1, 1, head_dim, group, bits, 16, 16,
                                       0, 0, 0, None)
    assert rc == _lib.KVX_ERR_INVALID_ARG
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_misaligned_pointers_rejected(lib):
    rc = lib.kvx_quant_pack(8, 16, 0, None, 1, 1, 1, 128, 128, 4, 16, 16, 16, 0, 0, 0, None)
    assert rc == _lib.KVX_ERR_INVALID_ARG


def test_head_window_out_of_range_rejected(lib):
    # window [3, 3+2) does not fit 4 heads per row
    rc = lib.kvx_quant_pack(256, 256, 0, None, 1, 1, 2, 128, 128, 4, 256, 256, 256, 0, 4, 3, None)
    assert rc == _lib.KVX_ERR_INVALID_ARG


def test_empty_is_a_noop(lib):
    assert lib.kvx_quant_pack(None, None, 0, None, 0, 0, 1, 128, 128, 4, None, None, None, 0,
                              0, 0, None) == 0
    assert lib.kvx_dequant_scatter_paged(None, None, None, 0, None, 4, 0, 8, 128, 128, 4, None,
                                         None, 0, 0, 0, None) == 0


def test_no_gpu_reports_zero_devices(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU host")
    n = ctypes.c_int(-1)
    assert lib.kvx_device_count(ctypes.byref(n)) == 0 and n.value == 0


def test_no_cpu_fallback(monkeypatch, tmp_path):
    """A missing extension must fail loudly, never fall back to the oracle."""
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load(str(tmp_path / "missing.so"))
    import glob
    pkg = os.path.join(ROOT, "paper_2502_09334_b200")
    for f in glob.glob(os.path.join(pkg, "*.py")):
        src = open(f).read()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f


def test_integration_doc_bindings_match():
    """The ctypes stub INTEGRATION.md shows a maintainer matches the real ABI."""
    src = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = {"P": ctypes.c_void_p, "I": ctypes.c_int, "I64": ctypes.c_int64, "U32": ctypes.c_uint32,
         "U64": ctypes.c_uint64, "PP": ctypes.POINTER(ctypes.c_void_p), "SZ": ctypes.c_size_t}
    found = re.findall(r"kvx\.(kvx_\w+)\.argtypes = \[([^\]]*)\]", src)
    assert len(found) >= 4
    for name, body in found:
        got = [m[x.strip()] for x in body.replace("\n", " ").split(",")]
        assert got == list(_lib.SIGNATURES[name]), name


def test_fused_and_kivi_entry_points_validate(lib):
    """The transport's fused kernels and the kivi pull variant reject bad
    arguments before touching CUDA (no GPU here)."""
    E = _lib.KVX_ERR_INVALID_ARG
    # K1 with doorbells: 16-bit has no doorbell variant; misaligned counters;
    # misaligned control block
    assert lib.kvx_quant_pack_signal(256, 256, 0, None, 1, 1, 1, 128, 128, 16, 256, 256, 256, 0,
                                     0, 0, 256, 256, 1, 1, None, 0, None, None) == E
    assert lib.kvx_quant_pack_signal(256, 256, 0, None, 1, 1, 1, 128, 128, 4, 256, 256, 256, 0,
                                     0, 0, 258, 256, 1, 1, None, 0, None, None) == E
    assert lib.kvx_quant_pack_signal(256, 256, 0, None, 1, 1, 1, 128, 128, 4, 256, 256, 256, 0,
                                     0, 0, 256, 256, 1, 1, None, 0, 260, None) == E
    # K3-bulk: in-kernel completion needs doorbells; unknown flags
    assert lib.kvx_pull_dequant_scatter_paged(256, 256, 256, 0, None, 1, 1, 1, 128, 128, 4, 256,
                                              256, 0, 0, 0, None, 1, 1, 256, 512, None, 0,
                                              None) == E
    assert lib.kvx_pull_dequant_scatter_paged(256, 256, 256, 0, None, 1, 1, 1, 128, 128, 4, 256,
                                              256, 0, 0, 0, 256, 1, 1, None, None, None, 4,
                                              None) == E
    # chained pulls only with programmatic dependent launch
    assert lib.kvx_pull_dequant_scatter_paged(256, 256, 256, 0, None, 1, 1, 1, 128, 128, 4, 256,
                                              256, 0, 0, 0, 256, 1, 1, None, None, None,
                                              _lib.KVX_PULL_CHAINED, None) == E
    offs = (ctypes.c_int64 * 7)(*([0] * 7))
    for fn in ("kvx_dequant_scatter_paged_kivi", "kvx_pull_dequant_scatter_paged_kivi"):
        f = getattr(lib, fn)
        tail = ((None,) if fn.startswith("kvx_dequant") else
                (None, 0, 1, None, None, None, 0, None))
        # kivi: bits 2 and group 128 are not kivi formats
        assert f(256, 256, offs, 256, None, 0, None, 0, 1, 1, 1, 128, 32, 2, 256, 256, 0,
                 *tail) == E
        assert f(256, 256, offs, 256, None, 0, None, 0, 1, 1, 1, 128, 128, 4, 256, 256, 0,
                 *tail) == E
        # group counts must add up to the token count
        assert f(256, 256, offs, 256, 256, 1, None, 0, 1, 5, 1, 128, 32, 4, 256, 256, 0,
                 *tail) == E
    # the pull variant's doorbells must be aligned
    assert lib.kvx_pull_dequant_scatter_paged_kivi(256, 256, offs, 256, None, 0, None, 0, 1, 32,
                                                   1, 128, 32, 4, 256, 256, 0, 258, 1, 1, None,
                                                   None, None, 0, None) == E
    # in-kernel slot release needs doorbells and both pointers (and, as
    # everywhere, group counts that add up to the token count)
    assert lib.kvx_pull_dequant_scatter_paged_kivi(256, 256, offs, 256, None, 0, None, 0, 1, 32,
                                                   1, 128, 32, 4, 256, 256, 0, None, 1, 1, 256,
                                                   256, None, 0, None) == E
    assert lib.kvx_pull_dequant_scatter_paged_kivi(256, 256, offs, 256, None, 0, 256, 1, 1, 32,
                                                   1, 128, 32, 4, 256, 256, 0, 256, 1, 1, 256,
                                                   256, None, 0, None) == E
    assert lib.kvx_pull_dequant_scatter_paged_kivi(256, 256, offs, 256, None, 0, None, 0, 1, 32,
                                                   1, 128, 32, 4, 256, 256, 0, 256, 1, 1, None,
                                                   None, None, 4, None) == E  # flags


def test_8bit_payload_stride_must_keep_32_byte_alignment(lib):
    """8-bit codes move as 32-byte vectors (st/ld.global.v8.b32): a payload
    layer stride that is a 16-byte but not a 32-byte multiple (48) would
    fault with a misaligned address on layer 1 -- the ABI rejects it."""
    E = _lib.KVX_ERR_INVALID_ARG
    # (k, v, src_ls, slots, L=2, T=1, H=1, D=128, G=128, bits, codes, scale, zero, stride, ...)
    assert lib.kvx_quant_pack(256, 256, 0, None, 2, 1, 1, 128, 128, 8, 256, 256, 256, 48, 0, 0,
                              None) == E
    assert lib.kvx_dequant_scatter_paged(256, 256, 256, 48, None, 2, 1, 1, 128, 128, 8, 256, 256,
                                         0, 0, 0, None) == E
    # 48 is fine at 4 bits (16-byte vectors): validation passes, the launch
    # then fails only for want of a GPU on this host
    rc = lib.kvx_quant_pack(256, 256, 0, None, 2, 1, 1, 128, 128, 4, 256, 256, 256, 48, 0, 0, None)
    assert rc != E
    # kivi: the 8-bit V codes (seg_offsets[4]) and the layer stride
    offs = (ctypes.c_int64 * 7)(0, 256, 512, 768, 1040, 2048, 2304)  # 1040 = 16 mod 32
    assert lib.kvx_quant_pack_kivi(256, 256, 0, 1, 32, 1, 128, 32, 8, 256, 1, None, 0, 256, 4096,
                                   offs, None) == E
    offs = (ctypes.c_int64 * 7)(0, 256, 512, 768, 1024, 2048, 2304)
    assert lib.kvx_quant_pack_kivi(256, 256, 0, 1, 32, 1, 128, 32, 8, 256, 1, None, 0, 256, 4112,
                                   offs, None) == E


def test_pair_entry_points_validate(lib):
    """kvx_pair_*: bad roles, formats, queue depths and alignments are
    rejected before any allocation (no GPU here); the chunk plan is pure."""
    E = _lib.KVX_ERR_INVALID_ARG
    out = ctypes.c_void_p()
    good = (0, 80, 4096, 8, 128, 4, 128, 2, 0, 4096, 8192, 1 << 20, 1 << 24, None)
    assert lib.kvx_pair_create(2, *good[1:], ctypes.byref(out)) == E      # role
    assert lib.kvx_pair_create(*good[:5], 16, *good[6:], ctypes.byref(out)) == E  # 16-bit
    assert lib.kvx_pair_create(*good[:7], 9, *good[8:], ctypes.byref(out)) == E   # Q > 8
    assert lib.kvx_pair_create(*good[:11], 4096 + 16, *good[12:], ctypes.byref(out)) == E  # queue
    assert lib.kvx_pair_create(*good[:13], 12, ctypes.byref(out)) == E   # ctl alignment
    assert lib.kvx_pair_send(None, 1, 256, 256, 0, None, 1, 0, 0, 0, None) == E
    assert lib.kvx_pair_recv(None, 1, 256, 256, 0, 256, 1, 0, 0, 0, None) == E
    slots = (ctypes.c_void_p * 1)(256)
    ns = (ctypes.c_int64 * 1)(16)
    assert lib.kvx_pair_recv_many(None, 1, 1, 256, 256, 0, slots, ns, 0, 0, 0, None) == E
    assert lib.kvx_pair_destroy(None) == 0
    lpc, nc = ctypes.c_int(), ctypes.c_int()
    # a 16-token 70B GQA hand-off is one chunk; config 3 is layer-granular
    assert lib.kvx_handoff_chunk_plan(80, 16, 8, 128, 0, ctypes.byref(lpc), ctypes.byref(nc)) == 0
    assert (lpc.value, nc.value) == (80, 1)
    assert lib.kvx_handoff_chunk_plan(40, 16384, 40, 128, 0, ctypes.byref(lpc),
                                      ctypes.byref(nc)) == 0
    assert (lpc.value, nc.value) == (1, 40)
    assert lib.kvx_handoff_chunk_plan(80, 16, 8, 128, 1, ctypes.byref(lpc), ctypes.byref(nc)) == 0
    assert (lpc.value, nc.value) == (2, 40)  # layer-wise: <= 64 chunks
    assert lib.kvx_handoff_chunk_plan(0, 16, 8, 128, 0, ctypes.byref(lpc), ctypes.byref(nc)) == E


def test_nccl_pool_entry_points(lib):
    """kvx_nccl_*: the paper's pre-built NCCL groups through the
    C-ABI.  Argument checks need no GPU; the unique id needs only NCCL's
    bootstrap (it is resolved at run time, no link-time dependency)."""
    E = _lib.KVX_ERR_INVALID_ARG
    assert lib.kvx_nccl_unique_id_size() == 128
    comm = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.kvx_nccl_pair_init(None, 2, 0, ctypes.byref(comm)) == E
    assert lib.kvx_nccl_pair_init(uid, 2, 2, ctypes.byref(comm)) == E
    assert lib.kvx_nccl_sendrecv(None, None, 0, -1, None, 0, -1, None) == E
    assert lib.kvx_nccl_sendrecv(256, None, 16, 1, None, 0, -1, None) == E
    assert lib.kvx_nccl_pair_destroy(None) == 0
    rc = lib.kvx_nccl_get_unique_id(uid)
    assert rc in (0, _lib.KVX_ERR_UNSUPPORTED, _lib.KVX_ERR_NCCL)
    if rc == 0:
        assert any(uid.raw)


def test_local_k3_choice_by_row_length(lib):
    """N=1 picks K3-bulk for rows of >= 64 chunks and the per-lane K3 for
    short rows (datapath.local_bulk_preferred; r02_bench/k3_local_geo_n1.log)."""
    from paper_2502_09334_b200.datapath import PackedLayout, local_bulk_preferred
    cfg2 = PackedLayout(32, 16384, 32, 128, 4, 128)    # 128 chunks per row
    cfg3 = PackedLayout(40, 16384, 40, 128, 8, 128)    # 160
    gqa = PackedLayout(80, 32768, 8, 128, 4, 128)      # 32: 70B-GQA, 8 KV heads
    raw = PackedLayout(32, 16384, 32, 128, 16, 128)    # passthrough
    assert local_bulk_preferred(cfg2) and local_bulk_preferred(cfg3)
    assert not local_bulk_preferred(gqa) and not local_bulk_preferred(raw)
