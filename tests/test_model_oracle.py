"""CPU tests for SURVEY 8(f) rows 1 and 4: the model-step oracle pinned against
reference-generated goldens, and the host-side training logic (schedule,
synthetic data, CSV writers) against the reference's own outputs."""

import csv
import io
import json
import os

import numpy as np
import pytest

from oracle import model_oracle as MO
from tests.conftest import GOLDEN

OPS = os.path.join(GOLDEN, "model_ops.npz")
TINY = os.path.join(GOLDEN, "model_tiny.npz")


@pytest.fixture(scope="module")
def ops():
    return np.load(OPS)


@pytest.fixture(scope="module")
def tiny():
    return np.load(TINY)


def test_rmsnorm_oracle_matches_reference(ops):
    y, r = MO.rmsnorm_fwd(ops["rms_x"], ops["rms_gain"])
    np.testing.assert_array_equal(y, ops["rms_y"])
    dx, dgain = MO.rmsnorm_bwd(ops["rms_x"], ops["rms_gain"], r, ops["rms_dy"])
    np.testing.assert_array_equal(dx, ops["rms_dx"])
    np.testing.assert_array_equal(dgain, ops["rms_dgain"])


def test_cross_entropy_oracle_matches_reference(ops):
    loss, p = MO.cross_entropy_fwd(ops["ce_logits"], ops["ce_targets"])
    assert loss == ops["ce_loss"]
    np.testing.assert_array_equal(MO.cross_entropy_bwd(p, ops["ce_targets"]), ops["ce_dlogits"])


def test_embedding_oracle_matches_reference(ops):
    np.testing.assert_array_equal(MO.embedding_fwd(ops["emb_table"], ops["emb_ids"]), ops["emb_out"])
    np.testing.assert_array_equal(MO.embedding_bwd(ops["emb_table"].shape, ops["emb_ids"], ops["emb_g"]),
                                  ops["emb_dtable"])


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_optimizer_oracle_is_bit_exact(ops, kind):
    for name in ("a", "b"):
        p = ops[f"opt_{kind}_{name}_p0"].copy()
        m = np.zeros_like(p)
        v = np.zeros_like(p)
        for step in range(3):
            g = ops[f"opt_{kind}_{name}_grads"][step]
            lr = 1e-3 * (step + 1)
            if kind == "adam":
                MO.adam_step(p, m, v, g, lr, step + 1)
            else:
                MO.sgd_step(p, m, g, lr)
            np.testing.assert_array_equal(p, ops[f"opt_{kind}_{name}_traj"][step])


def test_lr_schedule_matches_reference(ops):
    from paper_2412_09952_b200.train import Schedule, lr_at
    s = Schedule(lr_max=3e-3, lr_min=1e-4, warmup_steps=7, total_steps=50)
    got = np.array([lr_at(i, s) for i in ops["lr_steps"]])
    np.testing.assert_array_equal(got, ops["lr_values"])
    np.testing.assert_array_equal([MO.lr_at(i, 3e-3, 1e-4, 7, 50) for i in ops["lr_steps"]], ops["lr_values"])


def test_schedule_validation():
    from paper_2412_09952_b200.errors import ConfigError, InputError
    from paper_2412_09952_b200.train import Schedule, lr_at
    with pytest.raises(ConfigError):
        Schedule(1e-3, 2e-3, 1, 10)
    with pytest.raises(ConfigError):
        Schedule(1e-3, 1e-4, 10, 10)
    with pytest.raises(InputError):
        lr_at(11, Schedule(1e-3, 1e-4, 1, 10))


def test_synthetic_data_matches_reference(ops):
    from paper_2412_09952_b200.train import BlendSampler, BlendSpec, MarkovCorpus, _batch
    spec = BlendSpec((("a", 1.0), ("b", 2.0), ("c", 0.5)), seed=5)
    sampler = BlendSampler(spec)
    corpora = [MarkovCorpus(i, 96, spec.seed, 4) for i in range(3)]
    got = np.stack([_batch(corpora, sampler, 4, 17) for _ in range(3)])
    np.testing.assert_array_equal(got, ops["data_batches"])


def test_tiny_model_batch_is_the_reference_batch(tiny):
    from paper_2412_09952_b200.train import BlendSampler, BlendSpec, MarkovCorpus, _batch
    cfg = json.loads(str(tiny["config"]))
    spec = BlendSpec(tuple(tuple(s) for s in cfg["train"]["blend"][0]), cfg["train"]["blend"][1])
    sampler = BlendSampler(spec)
    corpora = [MarkovCorpus(i, cfg["model"]["vocab"], spec.seed, 4) for i in range(len(spec.sources))]
    tokens = _batch(corpora, sampler, cfg["train"]["batch_size"], cfg["train"]["seq_len"])
    np.testing.assert_array_equal(tokens, tiny["tokens"])


class _Stats:
    def __init__(self, drop_rate, assigned, gate_mass):
        self.drop_rate, self.assigned, self.gate_mass = drop_rate, np.array(assigned), np.array(gate_mass)


def test_routing_and_metrics_csv_text_match_reference(tiny, tmp_path):
    """Rebuild RunMetrics from the reference's CSV values and write them with
    this package's writers: the text must be byte-identical."""
    from paper_2412_09952_b200.train import METRICS_HEADER, RunMetrics
    rows = list(csv.reader(io.StringIO(str(tiny["routing_csv"]))))
    E = (len(rows[0]) - 3) // 2
    m = RunMetrics(run_id="tiny")
    mrows = list(csv.reader(io.StringIO(str(tiny["metrics_csv"]))))
    assert mrows[0] == METRICS_HEADER
    for r in mrows[1:]:
        m.steps.append(int(r[0]))
        m.loss.append(float(r[2]))
        m.lr.append(float(r[3]))
        m.drop_rate.append(float(r[4]))
        m.load_entropy.append(float(r[5]))
        m.layer_stats.append([])
    for r in rows[1:]:
        step = int(r[0])
        m.layer_stats[step].append(_Stats(float(r[2]), [int(a) for a in r[3:3 + E]],
                                          [float(g) for g in r[3 + E:3 + 2 * E]]))
    m.write_metrics_csv(str(tmp_path / "m.csv"))
    m.write_routing_csv(str(tmp_path / "r.csv"), E)
    assert (tmp_path / "m.csv").read_text() == str(tiny["metrics_csv"])
    assert (tmp_path / "r.csv").read_text() == str(tiny["routing_csv"])


def test_train_config_validation():
    from paper_2412_09952_b200.errors import ConfigError
    from paper_2412_09952_b200.train import BlendSpec, Schedule, TrainConfig
    s = Schedule(1e-3, 1e-4, 1, 5)
    b = BlendSpec((("a", 1.0),))
    with pytest.raises(ConfigError):
        TrainConfig(steps=0, schedule=s, blend=b)
    with pytest.raises(ConfigError):
        TrainConfig(steps=1, schedule=s, blend=b, optimizer="lion")
    with pytest.raises(ConfigError):
        BlendSpec((("a", -1.0),))


def test_moving_average_and_window_means():
    from paper_2412_09952_b200.train import moving_average, window_means
    v = [1.0, 2.0, 3.0, 4.0, 5.0]
    np.testing.assert_allclose(moving_average(v, 2), [1.5, 2.5, 3.5, 4.5])
    np.testing.assert_allclose(window_means(v, 2), [1.5, 3.5])


def test_model_symbols_exported():
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200 import _lib
    for name in ("forward_with_stats", "forward_logits", "train", "lr_at", "Schedule", "TrainConfig", "BlendSpec",
                 "eval_perplexity"):
        assert hasattr(P, name), name
    for sym in ("b200moe_rmsnorm_fwd", "b200moe_cross_entropy_bwd", "b200moe_optimizer_step"):
        assert sym in _lib.exported_symbols()
