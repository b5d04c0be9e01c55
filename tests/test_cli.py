"""CLI parity (cli.py:1-347, metrics.py:16-59) against
tests/golden/cli/golden.json, dumped from the reference's own CLI by
tests/golden/make_cli_golden.py.  gen, usage errors and the metrics record
are host-only (CPU tests); run / bench / the stage-wise commands call the
CUDA path (gpu)."""

import hashlib
import json
import os
import shutil

import pytest

from tests.golden_io import GOLDEN

CLI = os.path.join(GOLDEN, "cli")


def _golden():
    with open(os.path.join(CLI, "golden.json")) as f:
        return json.load(f)


def _sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def _record(path, base):
    d = json.loads(open(path).read().replace(str(base) + "/", ""))
    d.pop("stage_seconds", None)
    return d


@pytest.fixture
def work(tmp_path):
    for f in ("data.fvecs", "sparse.txt", "mixed.csv", "mixed.schema.json"):
        shutil.copy(os.path.join(CLI, f), tmp_path / f)
    return tmp_path


def test_gen_files_byte_identical(tmp_path):
    from paper_2106_10515_b200.cli import main

    p = lambda f: str(tmp_path / f)  # noqa: E731
    assert main(["gen", "--kind", "gaussian-mixture", "--n", "400", "--dim", "8", "--clusters", "5",
                 "--separation", "12", "--seed", "0", "--out", p("data.fvecs"), "--labels", p("labels.txt"),
                 "--meta", p("meta.json")]) == 0
    assert main(["gen", "--kind", "sparse-overlap", "--n", "120", "--dim", "4096", "--clusters", "4", "--seed", "3",
                 "--out", p("sparse.txt")]) == 0
    assert main(["gen", "--kind", "categorical-patterns", "--n", "90", "--dim", "6", "--clusters", "3",
                 "--seed", "5", "--out", p("cat.csv"), "--labels", p("cat_labels.txt")]) == 0
    for f, want in _golden()["gen_sha"].items():
        assert _sha(p(f)) == want, f


def test_usage_and_runtime_exit_codes(work):
    from paper_2106_10515_b200.cli import main

    g = _golden()
    base = {"data": str(work / "data.fvecs"), "data_kind": "dense", "metric": "jaccard", "workers": 1}
    (work / "bad.json").write_text(json.dumps(base))
    assert main(["run", "--config", str(work / "bad.json")]) == g["exit_bad_metric"] == 2
    (work / "nofile.json").write_text(json.dumps(dict(base, metric="euclidean", data=str(work / "nope.fvecs"))))
    assert main(["run", "--config", str(work / "nofile.json")]) == g["exit_missing_file"] == 1
    (work / "sp.json").write_text(json.dumps({"data": str(work / "sparse.txt"), "data_kind": "sparse",
                                              "metric": "euclidean", "workers": 1}))
    assert main(["run", "--config", str(work / "sp.json")]) == 2
    (work / "incomplete.json").write_text(json.dumps({"data": str(work / "data.fvecs")}))
    assert main(["run", "--config", str(work / "incomplete.json")]) == 2
    with pytest.raises(SystemExit) as e:
        main(["frobnicate"])
    assert e.value.code == 2


def test_metrics_record_roundtrip_and_reference_json():
    from paper_2106_10515_b200.metrics import MetricsRecord

    ref = dict(_golden()["run"]["2"], stage_seconds={"assign": 0.1})
    rec = MetricsRecord.from_json(json.dumps(ref))
    assert json.loads(rec.to_json()) == ref  # no `device` key unless populated
    rec.device = {"points_per_sec": 1.0}
    assert MetricsRecord.from_json(rec.to_json()) == rec
    rec.objective = float("nan")
    with pytest.raises(ValueError):
        rec.to_json()


@pytest.mark.gpu
def test_run_records_match_reference(work):
    from paper_2106_10515_b200.cli import main

    g = _golden()
    base = {"data": str(work / "data.fvecs"), "data_kind": "dense", "metric": "euclidean", "transform_tables": 8,
            "buckets_per_table": 20, "transform_seed": 1, "num_hashes": 3, "seeding_tables": 8,
            "min_group_size": 3, "seeding_seed": 2}
    for w in (1, 2):
        (work / f"run{w}.json").write_text(json.dumps(dict(base, workers=w)))
        assert main(["run", "--config", str(work / f"run{w}.json"), "--metrics", str(work / f"m{w}.json")]) == 0
        assert _record(work / f"m{w}.json", work) == g["run"][str(w)]
    # the device extension: counters and rates ride alongside the reference fields
    assert main(["run", "--config", str(work / "run2.json"), "--metrics", str(work / "md.json"),
                 "--device-metrics"]) == 0
    rec = json.loads((work / "md.json").read_text())
    dev = rec.pop("device")
    rec.pop("stage_seconds")
    assert json.loads(json.dumps(rec).replace(str(work) + "/", "")) == g["run"]["2"]
    assert dev["points_per_sec"] > 0 and "bucketize" in dev["phases"] and "split_boundary" in dev


@pytest.mark.gpu
def test_bench_grid_matches_reference(work):
    from paper_2106_10515_b200.cli import main

    cfg = {"data": str(work / "data.fvecs"), "data_kind": "dense", "metric": "euclidean", "workers": 1,
           "num_hashes": 3, "min_group_size": 3, "grid_t": [10, 20], "grid_m": [4, 8], "grid_L": [4, 8]}
    (work / "bench.json").write_text(json.dumps(cfg))
    assert main(["bench", "--config", str(work / "bench.json"), "--out", str(work / "out.jsonl")]) == 0
    got = [json.loads(line.replace(str(work) + "/", "")) for line in (work / "out.jsonl").read_text().splitlines()]
    for r in got:
        r.pop("stage_seconds")
    assert got == _golden()["bench"]


@pytest.mark.gpu
def test_stagewise_artifacts_match_reference(work):
    from paper_2106_10515_b200.cli import main

    g = _golden()
    p = lambda f: str(work / f)  # noqa: E731
    assert main(["transform", "--data", p("data.fvecs"), "--kind", "dense", "--tables", "8",
                 "--buckets-per-table", "20", "--seed", "1", "--out", p("buckets.bin")]) == 0
    assert main(["seed", "--buckets", p("buckets.bin"), "--universe", "400", "--num-hashes", "3", "--tables", "8",
                 "--min-group-size", "3", "--seed", "2", "--out", p("seeds.bin")]) == 0
    assert main(["assign", "--data", p("data.fvecs"), "--kind", "dense", "--seeds", p("seeds.bin"),
                 "--metric", "euclidean", "--out", p("clustering.bin"), "--metrics", p("ma.json")]) == 0
    for f, want in g["stage_sha"].items():
        assert _sha(p(f)) == want, f
    assert _record(p("ma.json"), work) == g["stage_record"]


@pytest.mark.gpu
def test_sparse_and_mixed_runs_match_reference(work):
    from paper_2106_10515_b200.cli import main

    g = _golden()
    p = lambda f: str(work / f)  # noqa: E731
    sp = {"data": p("sparse.txt"), "data_kind": "sparse", "metric": "jaccard", "workers": 2, "transform_tables": 4,
          "num_hashes": 2, "seeding_tables": 6, "min_group_size": 3, "target_dims": 256}
    (work / "sparse.json").write_text(json.dumps(sp))
    assert main(["run", "--config", p("sparse.json"), "--metrics", p("msp.json")]) == 0
    assert _record(p("msp.json"), work) == g["sparse"]
    mx = {"data": p("mixed.csv"), "data_kind": "mixed", "schema": p("mixed.schema.json"), "metric": "jaccard",
          "workers": 1, "transform_tables": 4, "num_hashes": 2, "seeding_tables": 4, "min_group_size": 2,
          "bins_per_attribute": 8}
    (work / "mixed.json").write_text(json.dumps(mx))
    assert main(["run", "--config", p("mixed.json"), "--metrics", p("mmx.json")]) == 0
    assert _record(p("mmx.json"), work) == g["mixed"]
    assert main(["transform", "--data", p("mixed.csv"), "--kind", "mixed", "--schema", p("mixed.schema.json"),
                 "--tables", "2", "--num-hashes", "2", "--seed", "1", "--bins-per-attribute", "8",
                 "--out", p("mxb.bin")]) == 0
    assert json.loads((work / "mxb.dictionaries.json").read_text()) == g["mixed_dicts"]
    assert _sha(p("mxb.bin")) == g["mixed_buckets_sha"]
