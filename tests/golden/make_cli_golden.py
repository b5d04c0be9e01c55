"""Golden outputs of the REAL reference CLI (lshclust.cli, cli.py:1-347) for
the CLI parity tests: generated files (gen), metrics records of run / bench /
the stage-wise commands (stage_seconds removed: wall-clock), artifact bytes.
Build container only:

    python tests/golden/make_cli_golden.py  ->  tests/golden/cli/*
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lshclust.cli import main  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def record(path):
    """a metrics record without its wall-clock field, file paths made relative"""
    d = json.loads(open(path).read().replace(OUT + "/", ""))
    d.pop("stage_seconds", None)
    return d


def main_():
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    g = {}
    p = lambda name: os.path.join(OUT, name)  # noqa: E731
    # gen: all three kinds
    assert main(["gen", "--kind", "gaussian-mixture", "--n", "400", "--dim", "8", "--clusters", "5",
                 "--separation", "12", "--seed", "0", "--out", p("data.fvecs"), "--labels", p("labels.txt"),
                 "--meta", p("meta.json")]) == 0
    assert main(["gen", "--kind", "sparse-overlap", "--n", "120", "--dim", "4096", "--clusters", "4", "--seed", "3",
                 "--out", p("sparse.txt")]) == 0
    assert main(["gen", "--kind", "categorical-patterns", "--n", "90", "--dim", "6", "--clusters", "3",
                 "--seed", "5", "--out", p("cat.csv"), "--labels", p("cat_labels.txt")]) == 0
    g["gen_sha"] = {f: sha(p(f)) for f in ("data.fvecs", "labels.txt", "meta.json", "sparse.txt", "cat.csv",
                                           "cat.schema.json", "cat_labels.txt")}
    # run (dense, g = 1 and 2)
    base = {"data": p("data.fvecs"), "data_kind": "dense", "metric": "euclidean", "transform_tables": 8,
            "buckets_per_table": 20, "transform_seed": 1, "num_hashes": 3, "seeding_tables": 8,
            "min_group_size": 3, "seeding_seed": 2}
    g["run"] = {}
    for w in (1, 2):
        cfg = dict(base, workers=w)
        json.dump(cfg, open(p(f"run{w}.json"), "w"))
        assert main(["run", "--config", p(f"run{w}.json"), "--metrics", p(f"m{w}.json")]) == 0
        g["run"][str(w)] = record(p(f"m{w}.json"))
    # bench grid
    bench = {"data": p("data.fvecs"), "data_kind": "dense", "metric": "euclidean", "workers": 1, "num_hashes": 3,
             "min_group_size": 3, "grid_t": [10, 20], "grid_m": [4, 8], "grid_L": [4, 8]}
    json.dump(bench, open(p("bench.json"), "w"))
    assert main(["bench", "--config", p("bench.json"), "--out", p("bench.jsonl")]) == 0
    g["bench"] = [{k: v for k, v in json.loads(line.replace(OUT + "/", "")).items() if k != "stage_seconds"}
                  for line in open(p("bench.jsonl")).read().strip().splitlines()]
    # stage-wise transform / seed / assign
    assert main(["transform", "--data", p("data.fvecs"), "--kind", "dense", "--tables", "8",
                 "--buckets-per-table", "20", "--seed", "1", "--out", p("buckets.bin")]) == 0
    assert main(["seed", "--buckets", p("buckets.bin"), "--universe", "400", "--num-hashes", "3", "--tables", "8",
                 "--min-group-size", "3", "--seed", "2", "--out", p("seeds.bin")]) == 0
    assert main(["assign", "--data", p("data.fvecs"), "--kind", "dense", "--seeds", p("seeds.bin"),
                 "--metric", "euclidean", "--out", p("clustering.bin"), "--metrics", p("ma.json")]) == 0
    g["stage_sha"] = {f: sha(p(f)) for f in ("buckets.bin", "seeds.bin", "clustering.bin")}
    g["stage_record"] = record(p("ma.json"))
    # sparse run
    sp = {"data": p("sparse.txt"), "data_kind": "sparse", "metric": "jaccard", "workers": 2, "transform_tables": 4,
          "num_hashes": 2, "seeding_tables": 6, "min_group_size": 3, "target_dims": 256}
    json.dump(sp, open(p("sparse.json"), "w"))
    assert main(["run", "--config", p("sparse.json"), "--metrics", p("msp.json")]) == 0
    g["sparse"] = record(p("msp.json"))
    # mixed CSV run + dictionaries
    rng = np.random.default_rng(0)
    rows = ["num,cat"] + [f"{rng.normal():.4f},c{rng.integers(0, 3)}" for _ in range(60)]
    open(p("mixed.csv"), "w").write("\n".join(rows) + "\n")
    json.dump({"columns": [{"name": "num", "kind": "numeric"}, {"name": "cat", "kind": "categorical"}]},
              open(p("mixed.schema.json"), "w"))
    mx = {"data": p("mixed.csv"), "data_kind": "mixed", "schema": p("mixed.schema.json"), "metric": "jaccard",
          "workers": 1, "transform_tables": 4, "num_hashes": 2, "seeding_tables": 4, "min_group_size": 2,
          "bins_per_attribute": 8}
    json.dump(mx, open(p("mixed.json"), "w"))
    assert main(["run", "--config", p("mixed.json"), "--metrics", p("mmx.json")]) == 0
    g["mixed"] = record(p("mmx.json"))
    assert main(["transform", "--data", p("mixed.csv"), "--kind", "mixed", "--schema", p("mixed.schema.json"),
                 "--tables", "2", "--num-hashes", "2", "--seed", "1", "--bins-per-attribute", "8",
                 "--out", p("mxb.bin")]) == 0
    g["mixed_dicts"] = json.loads(open(p("mxb.dictionaries.json")).read())
    g["mixed_buckets_sha"] = sha(p("mxb.bin"))
    # error exits
    bad = dict(base, workers=1, metric="jaccard")
    json.dump(bad, open(p("bad.json"), "w"))
    g["exit_bad_metric"] = main(["run", "--config", p("bad.json")])
    nofile = dict(base, workers=1, data=p("nope.fvecs"))
    json.dump(nofile, open(p("nofile.json"), "w"))
    g["exit_missing_file"] = main(["run", "--config", p("nofile.json")])
    # keep only what the tests read: inputs + golden.json (outputs are re-made by the test)
    keep = {"data.fvecs", "sparse.txt", "mixed.csv", "mixed.schema.json"}
    for f in os.listdir(OUT):
        if f not in keep:
            os.remove(p(f))
    json.dump(g, open(p("golden.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps({k: v for k, v in g.items() if k != "bench"}, indent=1)[:3000])


if __name__ == "__main__":
    main_()
