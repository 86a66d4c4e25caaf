"""The bench.py JSON line contract, checked on the committed round measurements
(profiles/r2_bench_*.json, written by bench.py on a B200): every key the driver
and the tier contract require, with the right types and units."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def line(name):
    path = os.path.join(PROF, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not committed")
    return json.loads(open(path).read().strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["r2_bench_default.json", "r2_bench_c5.json", "r2_bench_c1_graph.json"])
def test_bench_line_keys(name):
    d = line(name)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] >= 1 and d["steps"] >= 1 and d["warmup"] >= 3
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] < d["value"]
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and "reasons" in c
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"])


def test_bench_cpu_baseline_and_reference_arm():
    d = line("r2_bench_default.json")
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["unit"] == d["unit"]
    r = line("r2_bench_reference.json")
    assert r["impl"] == "reference" and r["unit"] == d["unit"] and r["metric"] == d["metric"]
    assert r["cpu_baseline"]["kind"] == "oracle"
    assert r["e2e"]["h2d_bytes_per_step"] == 0 and r["e2e"]["d2h_bytes_per_step"] == 0
    assert r["e2e"]["value"] == r["value"]
    # the oracle timed on the reported graph itself in the same run
    assert d["config"]["workload"] in cb["sample"] and cb["gpu_labels_bit_exact"] is True
    assert "secondary_sample" in cb and r["full_workload"]["value"] > 0


def test_byte_model_b_fin_terms():
    """bench.byte_model: the finish-phase bytes are SURVEY 8(d)'s B_fin for the implemented
    design -- its terms add up to the finish kernels' bytes; the full final compress adds
    exactly the 4n compress read (and drops the tile summaries / re-reads); second-level
    root checks (finish_gathers, h6_gathers) are never counted."""
    import numpy as np
    import bench
    n = 1 << 14
    ctr = {k: 0 for k in ("pending_links", "finish_vertices", "finish_edges", "sample_hooks", "finish_hooks",
                          "compress_writes", "h6_writes", "finish_gathers", "h6_gathers", "contract_roots")}
    ctr.update(pending_links=900, finish_vertices=7, finish_edges=55, finish_hooks=3, compress_writes=120,
               h6_writes=9, finish_gathers=10 ** 6, h6_gathers=10 ** 6, h6_tiles=2)
    lab = np.arange(n, dtype=np.uint32)
    Bp, xp = bench.byte_model((n // 2, n), n, 4 * n, 2, ctr, lab, lab, False, None, True)
    Bf, xf = bench.byte_model((n // 2, n), n, 4 * n, 2, ctr, lab, lab, False, None, False)
    tp, tf = xp["B_fin_terms"], xf["B_fin_terms"]
    assert sum(tp.values()) == Bp["finish_phase"]
    assert sum(tf.values()) == Bf["finish_phase"]
    assert Bf["finish_phase"] - Bp["finish_phase"] == (4 * n - (tp["tile_summaries"] - tf["tile_summaries"])
                                                       - tp["dirty_tile_rereads"])
    # the 10^6 second-level root checks appear nowhere in the bytes
    ctr2 = dict(ctr, finish_gathers=0, h6_gathers=0)
    assert bench.byte_model((n // 2, n), n, 4 * n, 2, ctr2, lab, lab, False, None, True)[0] == Bp
    assert xp["root_check_reads_not_counted"] == 2 * 10 ** 6
