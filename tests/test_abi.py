"""CPU-side checks of the C ABI boundary (no GPU compute): the library builds
for sm_100a, loads, exports every symbol include/nrc.h declares, validates
configs, and the host-only helpers agree with the paper readings."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nrc.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(nrc_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def libnrc():
    from paper_2106_12372_b200 import _lib
    return _lib.load()


def test_library_exports_every_declared_symbol(libnrc):
    from paper_2106_12372_b200 import _lib
    decl = declared_functions()
    assert len(decl) >= 20
    assert set(decl) == set(_lib.SYMBOLS)
    for name in decl:
        assert hasattr(libnrc, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.lib_path()], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(r"\bT " + name + r"\b", out), f"{name} not exported with C linkage"


def test_library_is_sm100a_tcgen05(libnrc):
    from paper_2106_12372_b200 import _lib
    sass = subprocess.run(["cuobjdump", "-sass", _lib.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.lib_path()], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "LDTM" in sass             # tcgen05.ld
    assert "UBLKCP" in sass           # TMA bulk copy
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


def _res_usage():
    """{kernel: registers}, {kernel: local-memory bytes} from cuobjdump -res-usage."""
    from paper_2106_12372_b200 import _lib
    out = subprocess.run(["cuobjdump", "-res-usage", _lib.lib_path()], capture_output=True, text=True).stdout
    rows = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) .*?LOCAL:(\d+)", out)
    return {f: int(r) for f, r, _ in rows}, {f: int(l) for f, _, l in rows}


def test_partials_kernel_fits_beside_an_optimiser_block(libnrc):
    """Co-residency budget (DESIGN 5.2): the next step's partials CTA becomes
    resident beside one optimiser block and gathers + encodes while the
    reduction runs.  Register files are split per SM sub-partition (16,384
    registers each); the partials CTA's 9 warps put 3 on one of them and an
    8-warp optimiser block 2, so 3 R_p + 2 R_a <= 512 (registers rounded up to
    8 per thread).  A partials kernel at 138 registers broke this and cost
    ~2 us per frame.  No hot kernel spills to local memory."""
    regs, local = _res_usage()
    up8 = lambda r: (int(r) + 7) // 8 * 8
    ra = up8(regs["_ZN3nrc17nrc_adam_w_kernelILi64EEEvNS_9AdamWArgsE"])
    for w in (32, 64):
        rp = up8(regs[f"_ZN3nrc19nrc_train_ws_kernelILi{w}ELb0EEEvNS_9TrainArgsE"])
        assert 3 * rp + 2 * ra <= 512, (w, rp, ra)
    for f, l in local.items():
        if "query_ts_kernel" in f or "train_ws_kernel" in f or "adam_w_kernel" in f:
            assert l == 0, f


def test_default_config_and_state_bytes(libnrc):
    from paper_2106_12372_b200 import _lib
    c = _lib.NrcConfig()
    libnrc.nrc_default_config(ctypes.byref(c))
    assert c.abi_version == 2 and c.hidden_width == 64 and c.n_hidden_layers == 5
    assert c.loss_eps == pytest.approx(0.01) and c.ema_alpha == pytest.approx(0.99)
    assert c.learning_rate == pytest.approx(1e-2) and c.flags == 3
    nb = libnrc.nrc_state_bytes(ctypes.byref(c))
    assert nb > 21504 * 4 * 4 + 2 * 43008
    bad = _lib.NrcConfig(); libnrc.nrc_default_config(ctypes.byref(bad)); bad.hidden_width = 96
    assert libnrc.nrc_state_bytes(ctypes.byref(bad)) == 0
    bad.hidden_width = 64; bad.aabb_max[1] = bad.aabb_min[1]
    assert libnrc.nrc_state_bytes(ctypes.byref(bad)) == 0
    bad.aabb_max[1] = 1.0; bad.abi_version = 7
    assert libnrc.nrc_state_bytes(ctypes.byref(bad)) == 0
    bad.abi_version = 2; bad.max_batch = 0
    assert libnrc.nrc_state_bytes(ctypes.byref(bad)) == 0
    bad.max_batch = 3840 * 2160 * 4  # 64-bit max_batch beyond 2^32 is accepted
    bad.max_batch = 2 ** 33
    assert libnrc.nrc_state_bytes(ctypes.byref(bad)) == nb


def test_config_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of nrc_config has the C struct's size and field
    offsets (compiled from include/nrc.h with the host compiler)."""
    from paper_2106_12372_b200 import _lib
    fields = [f for f, _ in _lib.NrcConfig._fields_]
    src = tmp_path / "off.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"nrc.h\"\nint main(void){\n"
                   + f'printf("%zu\\n", sizeof(nrc_config));\n'
                   + "".join(f'printf("%zu\\n", offsetof(nrc_config, {f}));\n' for f in fields) + "return 0;}\n")
    exe = tmp_path / "off"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got[0] == ctypes.sizeof(_lib.NrcConfig)
    assert got[1:] == [getattr(_lib.NrcConfig, f).offset for f in fields]


def test_init_rejects_bad_arguments_without_gpu(libnrc):
    from paper_2106_12372_b200 import _lib
    c = _lib.NrcConfig(); libnrc.nrc_default_config(ctypes.byref(c))
    h = ctypes.c_void_p()
    assert libnrc.nrc_init(ctypes.byref(c), None, 0, ctypes.byref(h)) == 1  # NULL state
    assert libnrc.nrc_query(None, None, 0, None, None) == 6                 # NULL handle -> STATE
    assert libnrc.nrc_status_string(0) == b"NRC_OK"
    assert libnrc.nrc_param_count(None) == 20672


def test_lcg_params_match_oracle(libnrc, orc):
    # both sides implement reading R15 independently; the constants must agree
    from paper_2106_12372_b200 import lcg_params
    for n in (1, 2, 3, 1000, 16384, 65536, 65537, 2 ** 20):
        for seed in (0, 7, 0xFFFFFFFFFFFF):
            assert lcg_params(n, seed) == orc.lcg_params(n, seed)


def test_frame_scratch_bytes(libnrc):
    assert libnrc.nrc_frame_scratch_bytes(0, 0) >= 0
    nb = libnrc.nrc_frame_scratch_bytes(2073600, 65536)
    assert nb >= 2073600 * (64 + 12) + 65536 * 76


@pytest.mark.parametrize("hw,nh,ok", [(64, 5, True), (64, 1, True), (64, 7, True), (64, 8, False), (64, 0, False),
                                      (32, 8, True), (32, 9, False), (128, 5, True), (128, 6, False)])
def test_state_bytes_depth_and_width(libnrc, hw, nh, ok):
    """Host-side sizing of the state arena for the width / depth variants
    (SURVEY C4, N4): the arena holds the four fp32 parameter arrays of the
    padded layout (64 W + (n-1) W^2 + 16 W floats), two fp16 operand images
    and 256 per-CTA fp32 gradient partials; unsupported depths give 0."""
    from paper_2106_12372_b200 import _lib
    c = _lib.NrcConfig(); libnrc.nrc_default_config(ctypes.byref(c))
    c.hidden_width, c.n_hidden_layers = hw, nh
    nb = libnrc.nrc_state_bytes(ctypes.byref(c))
    if not ok:
        assert nb == 0
        return
    padded = 64 * hw + (nh - 1) * hw * hw + 16 * hw
    assert nb >= 4 * 4 * padded + 256 * 4 * padded
    # one more hidden layer adds W^2 floats to every per-parameter array
    if nh > 1:
        c.n_hidden_layers = nh - 1
        assert libnrc.nrc_state_bytes(ctypes.byref(c)) < nb


def test_nvls_entry_points_validate_arguments(libnrc):
    """nrc_train_apply_multimem / nrc_peer_barrier / nrc_multicast_alloc reject
    bad arguments without touching a GPU, and the multimem.ld_reduce load of
    the NVLS optimiser is in the binary (LDGMC)."""
    from paper_2106_12372_b200 import _lib
    STATE, INVALID = 6, 1
    assert libnrc.nrc_train_apply_multimem(None, None, 1, None, None) == STATE
    assert libnrc.nrc_peer_barrier(None, None, 0, 1, None) == STATE
    uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
    assert libnrc.nrc_multicast_alloc(0, 0, ctypes.byref(uc), ctypes.byref(mc)) == INVALID
    assert libnrc.nrc_multicast_alloc(0, 1024, None, ctypes.byref(mc)) == INVALID
    assert libnrc.nrc_multicast_free(None) == INVALID
    sass = subprocess.run(["cuobjdump", "-sass", _lib.lib_path()], capture_output=True, text=True).stdout
    assert "LDGMC" in sass  # multimem.ld_reduce (NVLS all-reduce read by the optimiser)
