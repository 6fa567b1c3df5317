"""The C ABI consumed from plain C99 (tests/c/abi_consumer.c): the header compiles with
`gcc -std=c99 -pedantic`, the program links libnestrack.so and drives the builder, and the
struct layouts the compiler computes equal the Python ctypes mirrors field by field."""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def consumer(tmp_path_factory):
    from paper_2406_13849_b200 import build as nb
    nb.build()
    exe = str(tmp_path_factory.mktemp("c") / "abi_consumer")
    libdir = os.path.join(ROOT, "paper_2406_13849_b200")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror",
                           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "abi_consumer.c"),
                           "-L", libdir, "-lnestrack", f"-Wl,-rpath,{libdir}", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


def _mirror(cls):
    return {name: getattr(cls, name).offset for name, _ in cls._fields_}


@pytest.mark.parametrize("cname,pyname", [("nt_build_opts", "BuildOpts"), ("nt_model_info", "ModelInfo"),
                                          ("nt_run", "Run"), ("nt_outputs", "Outputs")])
def test_struct_layouts_match_ctypes(consumer, cname, pyname):
    import paper_2406_13849_b200 as nt
    cls = getattr(nt, pyname)
    assert consumer[f"sizeof.{cname}"] == C.sizeof(cls)
    offs = _mirror(cls)
    checked = 0
    for key, val in consumer.items():
        if key.startswith(cname + "."):
            field = key.split(".", 1)[1]
            assert offs[field] == val, (cname, field, offs[field], val)
            checked += 1
    assert checked >= 5


def test_trace_record_layout(consumer):
    import oracle
    import paper_2406_13849_b200 as nt
    for dt in (nt.TRACE_DTYPE, oracle.TRACE_DTYPE):
        assert consumer["sizeof.nt_trace_rec"] == dt.itemsize
        for f in dt.names:
            assert consumer[f"nt_trace_rec.{f}"] == dt.fields[f][1], f


def test_builder_and_errors_from_c(consumer):
    assert consumer["abi_version"] == 4
    assert consumer["n_surfaces"] == 9 and consumer["n_cells"] == 5 and consumer["n_material_cells"] == 4
    assert consumer["max_depth"] == 2 and consumer["rect_specialisable"] == 1
    assert consumer["out_len"] == 2 * 4 + 18
    assert consumer["add_after_finalize"] == -3               # NT_E_ORDER
    assert consumer["track_host_only"] == -3 and "host-only" in consumer["track_host_only_msg"]
    assert consumer["bad_kind"] == -1                         # NT_E_ARG
    assert consumer["bad_material"] == 0 and consumer["bad_material_finalize"] == -4   # NT_E_GEOMETRY
    assert np.isfinite(consumer["sizeof.nt_run"])
