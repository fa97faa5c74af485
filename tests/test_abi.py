"""Host-side checks of the C-ABI library (no GPU needed): it builds for sm_100a, loads,
and exports every entry point include/snn.h declares; the binding has the same names;
the product path never imports the oracle."""
import ast
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2212_07679_b200 import build_lib
    return build_lib.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "snn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(snn_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ["snn_build", "snn_query_radius", "snn_free"]:   # BASELINE.json north_star
        assert f in fns


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for f in header_functions():
        assert hasattr(lib, f), f
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath]).decode()
    exported = set(re.findall(r" T (snn_\w+)", out))
    assert set(header_functions()) <= exported


def test_library_is_sm100a_only(libpath):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath]).decode()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_sass_uses_bulk_async_copy(libpath):
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath]).decode()
    assert "UBLKCP" in sass     # cp.async.bulk (TMA engine) staging of candidate rows


def test_k8_two_query_step_loop_has_no_fp64(libpath):
    """The K8 two-queries-per-thread scan (window_lowd_2q, default for 2 <= d <= 8): ptxas once
    rematerialised the fp64 filter threshold inside the step loop (12 fp64 instructions per
    step, DESIGN.md section 6 'the binding resource').  The loop -- from its first LDS.128
    to the warp vote that closes a step -- must hold packed FP32 FMAs and no fp64."""
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath]).decode()
    fns = re.split(r"\n\s*Function : ", sass)
    seen = 0
    for fn in fns:
        name = fn.split("\n", 1)[0]
        m = re.search(r"window_lowd_2qILi([23])ELb[01]E", name)
        if not m:
            continue
        ops = [re.sub(r"^@!?U?P\d+\s+", "", x) for x in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", fn)]
        first = next(i for i, o in enumerate(ops) if o.startswith("LDS.128"))
        vote = next(i for i in range(first, len(ops)) if ops[i].startswith("VOTE.ANY"))
        loop = ops[first:vote]
        nf = sum(o.startswith("FFMA2") for o in loop)   # 8 d packed FMAs per step (2 queries x 8 candidates)
        assert nf > 0 and nf % (8 * int(m.group(1))) == 0, name
        assert not [o for o in loop if re.match(r"D(FMA|MUL|ADD)|F2F", o)], name
        seen += 1
    assert seen >= 4


def test_binding_names_match_header():
    import paper_2212_07679_b200 as p
    for f in header_functions():
        assert hasattr(p, f), f
    assert sorted(p.EXPORTS) == sorted(header_functions())


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2212_07679_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names)
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle")
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                for line in open(os.path.join(dirpath, f)):
                    if line.strip().startswith("#include"):
                        assert "oracle" not in line.lower()


def test_missing_library_fails_loudly(tmp_path):
    import paper_2212_07679_b200 as p
    saved = p._lib
    try:
        p._lib = None
        with pytest.raises(RuntimeError, match="CUDA library missing"):
            p.load_library(str(tmp_path / "nope.so"))
    finally:
        p._lib = saved


def test_snn_load_rejects_bad_files_without_touching_the_device(libpath, tmp_path):
    """snn_load validates magic, version, header and length on the host first (the SPEC
    io_persist error cases) -- runnable without a GPU."""
    import struct
    import paper_2212_07679_b200 as p
    p.load_library()
    hdr = [5, 8, 2, 0, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0] + [0] * 8   # n=5, n_pad=8, d=2, ld=0, f32, euclidean
    cases = {
        "bad magic": b"XXXX" + struct.pack("<I", 1) + struct.pack("<23q", *hdr),
        "unsupported version": b"SNNG" + struct.pack("<I", 2) + struct.pack("<23q", *hdr),
        "truncated": b"SNNG" + struct.pack("<I", 1) + struct.pack("<23q", *hdr)[:40],
        "invalid header": b"SNNG" + struct.pack("<I", 1) + struct.pack("<23q", *([5, 7] + hdr[2:])),
        "invalid header ": b"SNNG" + struct.pack("<I", 1) + struct.pack("<23q", *(hdr[:3] + [3] + hdr[4:])),
    }
    # correct header, payload one byte short
    cases["truncated "] = cases["unsupported version"][:4] + struct.pack("<I", 1) + \
        struct.pack("<23q", *hdr) + b"\0" * 100
    for want, blob in cases.items():
        f = tmp_path / "x.snn"
        f.write_bytes(blob)
        with pytest.raises(p.SnnError, match=want.strip()):
            p.snn_load(str(f))
    with pytest.raises(p.SnnError, match="cannot open"):
        p.snn_load(str(tmp_path / "missing.snn"))


def test_header_is_plain_c(tmp_path):
    """include/snn.h compiles as C99 and as C++17 on its own (no torch / CUDA types in the
    boundary)."""
    src = tmp_path / "h.c"
    src.write_text('#include "include/snn.h"\nint main(void) { return 0; }\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I", ROOT, str(src)])
    subprocess.check_call(["g++", "-std=c++17", "-Wall", "-Werror", "-fsyntax-only", "-x", "c++", "-I", ROOT, str(src)])


def test_c_demo_links_against_the_library(libpath, tmp_path):
    """examples/c_api_demo.c (plain C99, no CUDA headers) compiles and links against
    lib/libsnn.so: the boundary is usable without Python."""
    exe = tmp_path / "c_api_demo"
    libdir = os.path.dirname(libpath)
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", libdir, "-lsnn",
                           f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    assert exe.exists()


def test_options_are_per_thread(libpath):
    """snn_set_option changes only the calling thread's options (include/snn.h): a second
    thread starts from the defaults and its changes do not leak back (no GPU needed)."""
    import threading
    import paper_2212_07679_b200 as p
    p.load_library()
    p.snn_set_option("tc_tiles", 4)
    seen = {}

    def other():
        seen["tc_tiles"] = p.snn_get_option("tc_tiles")
        p.snn_set_option("chunk", 1024)
        seen["chunk"] = p.snn_get_option("chunk")
    try:
        t = threading.Thread(target=other)
        t.start()
        t.join()
        assert seen == {"tc_tiles": 8, "chunk": 1024}
        assert p.snn_get_option("tc_tiles") == 4 and p.snn_get_option("chunk") == 2048
        with pytest.raises(p.SnnError, match="unknown option"):
            p.snn_get_option("no_such_option")
    finally:
        p.snn_set_option("tc_tiles", 0)
    assert p.snn_get_option("tc_tiles") == 8
