"""Load the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


@functools.lru_cache(maxsize=None)
def _load(name: str):
    z = np.load(os.path.join(GOLDEN, name))
    data = {k: z[k] for k in z.files}
    meta = json.loads(bytes(data.pop("meta")).decode())
    return data, meta


def step_cases():
    data, meta = _load("golden_steps.npz")
    return meta["cases"]


def step_sizes():
    _, meta = _load("golden_steps.npz")
    return {k: tuple(v) for k, v in meta["sizes"].items()}


def step_case(name: str) -> dict:
    """Structured view of one step case: inputs per rank, reference outputs."""
    data, meta = _load("golden_steps.npz")
    case = next(c for c in meta["cases"] if c["name"] == name)
    sizes = step_sizes()
    world = case["world"]
    p = f"{name}/"
    out = dict(case=case, sizes=sizes,
               theta={k: data[p + f"in/theta/{k}"] for k in sizes},
               m=[{k: data[p + f"in/m/{r}/{k}"] for k in sizes} for r in range(world)],
               g=[{k: data[p + f"in/g/{r}/{k}"] for k in sizes} for r in range(world)],
               theta_out={k: data[p + f"out/theta/{k}"] for k in sizes},
               m_out=[{k: data[p + f"out/m/{r}/{k}"] for k in sizes} for r in range(world)],
               sign={k: data[p + f"out/sign/{k}"].astype(np.int64) for k in sizes},
               ties={k: int(data[p + f"out/ties/{k}"]) for k in sizes},
               words=[{k: data.get(p + f"out/words/{r}/{k}") for k in sizes}
                      for r in range(world)],
               q=[{k: data.get(p + f"out/q/{r}/{k}") for k in sizes} for r in range(world)],
               norm=[{k: data.get(p + f"out/norm/{r}/{k}") for k in sizes}
                     for r in range(world)],
               c=[{k: data.get(p + f"out/c/{r}/{k}") for k in sizes} for r in range(world)],
               agree=data.get(p + "out/agree"), timing_keys=data.get(p + "out/timing_keys"),
               mask={k: data[p + f"in/mask/{k}"] for k in sizes
                     if (p + f"in/mask/{k}") in data} or None)
    return out


def collective_cases():
    _, meta = _load("golden_collectives.npz")
    return meta["cases"]


def collective_case(name: str) -> dict:
    data, meta = _load("golden_collectives.npz")
    case = next(c for c in meta["cases"] if c["name"] == name)
    p = f"{name}/"
    return dict(case=case,
                inputs=[data[p + f"in/{r}"] for r in range(case["world"])],
                values=data[p + "out/values"],
                ties=int(data[p + "out/ties"]) if (p + "out/ties") in data else None)


def quant_golden():
    """golden_quant.npz: the reference's standalone quant.py outputs."""
    return _load("golden_quant.npz")


def metrics_golden():
    """golden_metrics.npz: the reference's signsgd_majority_step and
    momentum-divergence outputs."""
    return _load("golden_metrics.npz")


def signsgd_case(i: int, sizes: dict):
    data, meta = metrics_golden()
    algo, world, kind, zm, it = meta["signsgd"][i]
    p = f"sgd{i}/"
    return dict(
        algo=algo, world=world, zero_mode=zm, iteration=it,
        theta={k: data[p + f"in/theta/{k}"] for k in sizes},
        m=[{k: data[p + f"in/m/{r}/{k}"] for k in sizes} for r in range(world)],
        g=[{k: data[p + f"in/g/{r}/{k}"] for k in sizes} for r in range(world)],
        theta_out={k: data[p + f"out/theta/{k}"] for k in sizes},
        div={k: float(data[p + f"out/div/{k}"]) for k in sizes},
        divm={k: float(data[p + f"out/divm/{k}"]) for k in sizes})
