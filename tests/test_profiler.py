"""Measured install phase (runtime/profiler.py): grid coverage, entry semantics and
the shardplan-profile v1 round trip, with a fake kernel bench on CPU; the real
kernels on the B200 under -m gpu."""

import math

import pytest

from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.planning.costdb import (Generator, KernelKey, estimate_kernel_time, grid_shapes,
                                                   load_profile, lookup_exact, save_profile, synth_profile)
from paper_2604_26334_b200.planning.placement import plan_tier
from paper_2604_26334_b200.planning.vocab import Backend, OpKind, canonical_workload
from paper_2604_26334_b200.runtime import profiler


class FakeBench:
    """Deterministic stand-in: time = 1 us + bytes / 5 TB/s + flops / 1 PF/s."""

    torch = None

    def run(self, op, dims):
        flops, byts = canonical_workload(op, dims, 2.0)
        return "fake", 1e-6 + byts / 5e12 + flops / 1e15


def test_measured_profile_replaces_only_f16_gpu_entries(tmp_path):
    machine = catalog.builtin_machine("b200")
    points = profiler.measure_points(bench=FakeBench())
    assert len(points) == len(grid_shapes())
    db = profiler.measured_profile(machine, points)
    synth = synth_profile(machine)
    assert len(db) == len(synth)
    assert db.meta.generator is Generator.MEASURED
    changed = 0
    for e, s in zip(db.entries(), synth.entries()):
        assert e.key == s.key
        if e.key.backend is Backend.GPU and e.key.quant == "f16":
            changed += 1
            flops, byts = canonical_workload(e.key.op_kind, e.key.dims, 2.0)
            secs = FakeBench().run(e.key.op_kind, e.key.dims)[1]
            # an exact hit returns the measured time
            t, kind = estimate_kernel_time(db, e.key, flops, byts)
            assert math.isclose(t, secs, rel_tol=1e-12)
        else:
            assert (e.flops_per_sec, e.bytes_per_sec) == (s.flops_per_sec, s.bytes_per_sec)
    assert changed == len(grid_shapes())
    path = tmp_path / "m.profile"
    save_profile(db, path)
    back = load_profile(path)
    assert back.meta.generator is Generator.MEASURED
    assert [(e.key, e.flops_per_sec, e.bytes_per_sec) for e in back.entries()] == \
        [(e.key, e.flops_per_sec, e.bytes_per_sec) for e in db.entries()]
    profiler.write_sidecar(str(tmp_path / "m.json"), machine, points)


def test_planner_runs_on_a_measured_profile():
    machine = catalog.builtin_machine("b200")
    db = profiler.measured_profile(machine, profiler.measure_points(bench=FakeBench()))
    spec = catalog.builtin_model("llama3.1-8b")
    _shards, _pin, _split, plans = plan_tier(spec, machine, db, 4e9, 2304, 1)
    assert all(p.estimated_time > 0 for p in plans if p.feasible)
    key = KernelKey(OpKind.MATMUL, "f16", Backend.GPU, 0, (1, 4096, 4096))
    assert lookup_exact(db, key) is not None


@pytest.mark.gpu
def test_real_kernels_on_a_grid_subset():
    """Every op kind through its real kernel; achieved rates must be physical
    (below 1.3x the measured copy / GEMM peaks)."""
    shapes = [(OpKind.MATMUL, (1, 4096, 16384)), (OpKind.MATMUL, (2048, 4096, 4096)),
              (OpKind.GQA, (1, 16384, 32, 8, 128)), (OpKind.GQA, (512, 1024, 32, 8, 128)),
              (OpKind.MHA, (4, 1024, 32, 128)), (OpKind.MOE_ROUTE, (1, 2048, 128)),
              (OpKind.MOE_ROUTE, (1024, 2048, 128)), (OpKind.ELEMENT_WISE, (1 << 24,))]
    points = profiler.measure_points(shapes)
    for p in points:
        assert p.seconds > 0
        assert p.bytes / p.seconds < 1.3 * 6.6e12, p
        assert p.flops / p.seconds < 1.3 * 2.25e15, p
    gemv = points[0]
    assert gemv.bytes / gemv.seconds > 2e12, gemv   # a 128 MB GEMV streams at HBM rates
    gemm = points[1]
    assert gemm.flops / gemm.seconds > 5e14, gemm   # tcgen05 GEMM
