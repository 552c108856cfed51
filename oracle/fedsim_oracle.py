"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

float64 NumPy restatement of the reference's device-side hot path
(``/root/reference/pkg/src/fedsim``, abbreviated ``fedsim/`` below).  It is the
checker the CUDA path is compared against; it is pinned against golden
vectors produced by running the reference itself (tests/golden/).

Models are flat dicts ``{name: float64 ndarray}``; a "result" is a dict
``{name: (tensor, op, weight, client_id)}`` with ``op`` one of the strings
"WeightedAverage", "Sum", "SimpleAverage", "Collect" (fedsim/trainer.py:35-39).
"""

from __future__ import annotations

import numpy as np

WA, SUM, SA, COLLECT = "WeightedAverage", "Sum", "SimpleAverage", "Collect"
STREAM_SELECTION, STREAM_MINIBATCH, STREAM_NOISE, STREAM_SCHEDULE = 1, 6, 4, 5


# ---------------------------------------------------------------------------
# RNG streams and selection  (fedsim/core.py:22-32, :178-187)
# ---------------------------------------------------------------------------

def rng_for(seed: int, stream: int, *ctx: int) -> np.random.Generator:
    """fedsim/core.py:30-32 -- PCG64 seeded by SeedSequence([seed, stream, *ctx])."""
    return np.random.default_rng([seed, stream, *ctx])


def selection(seed: int, total: int, per_round: int, rnd: int) -> list[int]:
    """fedsim/core.py:178-187 -- uniform without replacement, draw order kept."""
    drawn = rng_for(seed, STREAM_SELECTION, rnd).choice(total, size=per_round,
                                                        replace=False)
    return [int(v) for v in drawn]


def minibatch_orders(seed: int, client_id: int, rnd: int, n: int,
                     epochs: int) -> list[np.ndarray]:
    """fedsim/trainer.py:445,452-453 -- one permutation of range(n) per epoch,
    all drawn from the (seed, 6, client, round) stream in epoch order."""
    g = rng_for(seed, STREAM_MINIBATCH, client_id, rnd)
    return [g.permutation(n) for _ in range(epochs)]


# ---------------------------------------------------------------------------
# Multinomial logistic regression  (fedsim/trainer.py:124-158)
# ---------------------------------------------------------------------------

def _shifted_logits(W, b, X):
    """fedsim/trainer.py:124-128: z - max(z), and log-sum-exp of the shifted z."""
    z = X @ W.T + b
    z = z - z.max(axis=1, keepdims=True)
    return z, np.log(np.exp(z).sum(axis=1))


def ce_loss(W, b, X, y) -> float:
    """fedsim/trainer.py:131-133."""
    z, lse = _shifted_logits(W, b, X)
    return float(np.mean(lse - z[np.arange(len(y)), y]))


def ce_loss_grad(W, b, X, y):
    """fedsim/trainer.py:136-145: mean CE and (P - onehot)^T X / B, sum(P - onehot)/B."""
    z, lse = _shifted_logits(W, b, X)
    rows = np.arange(len(y))
    loss = float(np.mean(lse - z[rows, y]))
    delta = np.exp(z - lse[:, None])
    delta[rows, y] -= 1.0
    delta /= len(y)
    return loss, delta.T @ X, delta.sum(axis=0)


def accuracy_and_loss(W, b, X, y) -> tuple[float, float]:
    """fedsim/trainer.py:148-158."""
    z, lse = _shifted_logits(W, b, X)
    return (float(np.mean(z.argmax(axis=1) == y)),
            float(np.mean(lse - z[np.arange(len(y)), y])))


# ---------------------------------------------------------------------------
# Algorithm plugins  (fedsim/trainer.py:172-424)
# ---------------------------------------------------------------------------

class Algo:
    """Hyper-parameters of one reference plugin (fedsim/trainer.py:185-191,
    :243-247, :303-307, :359-366)."""

    def __init__(self, name: str, lr: float = 0.1, batch_size: int = 0,
                 mu: float = 0.01, alpha: float = 0.1,
                 client_fraction: float = 1.0, collect_local_loss: bool = False):
        self.name, self.lr, self.batch_size = name.lower(), float(lr), int(batch_size)
        self.mu, self.alpha = float(mu), float(alpha)
        self.client_fraction = float(client_fraction)
        self.collect_local_loss = bool(collect_local_loss)

    @property
    def stateful(self) -> bool:
        return self.name in ("scaffold", "feddyn")

    # fedsim/trainer.py:193-197, :309-313, :368-374
    def init_global(self, W, b) -> dict:
        W, b = np.asarray(W, float), np.asarray(b, float)
        if self.name == "feddyn":
            return {"weights": (W.copy(), SA), "bias": (b.copy(), SA),
                    "server_h_weights": (np.zeros_like(W), SUM),
                    "server_h_bias": (np.zeros_like(b), SUM)}
        g = {"weights": (W.copy(), WA), "bias": (b.copy(), WA)}
        if self.name == "scaffold":
            g["server_ctrl_weights"] = (np.zeros_like(W), SUM)
            g["server_ctrl_bias"] = (np.zeros_like(b), SUM)
        return g

    # fedsim/trainer.py:315-317, :376-378
    def default_state(self, W, b):
        if self.name == "scaffold":
            return {"ctrl_weights": np.zeros_like(W), "ctrl_bias": np.zeros_like(b)}
        if self.name == "feddyn":
            return {"grad_corr_weights": np.zeros_like(W),
                    "grad_corr_bias": np.zeros_like(b)}
        return None

    def gradient(self, W, b, X, y, W0, b0, glob, state):
        """local_gradient hooks: fedsim/trainer.py:223-224 (FedAvg/FedNova),
        :249-257 (FedProx), :319-323 (SCAFFOLD), :380-386 (FedDyn)."""
        loss, gW, gb = ce_loss_grad(W, b, X, y)
        if self.name == "fedprox" and self.mu != 0.0:
            dW, db = W - W0, b - b0
            loss += 0.5 * self.mu * (float(np.sum(dW * dW)) + float(np.sum(db * db)))
            gW, gb = gW + self.mu * dW, gb + self.mu * db
        elif self.name == "scaffold":
            gW = gW + (glob["server_ctrl_weights"][0] - state["ctrl_weights"])
            gb = gb + (glob["server_ctrl_bias"][0] - state["ctrl_bias"])
        elif self.name == "feddyn":
            gW = gW - state["grad_corr_weights"] + self.alpha * (W - W0)
            gb = gb - state["grad_corr_bias"] + self.alpha * (b - b0)
        return loss, gW, gb

    def finalize(self, W, b, steps, W0, b0, glob, state, n):
        """fedsim/trainer.py:226-230, :268-278, :325-338, :388-395."""
        if self.name in ("fedavg", "fedprox"):
            return {"weights": (W, WA, float(n), None),
                    "bias": (b, WA, float(n), None)}, None
        if self.name == "fednova":
            scale = self.lr * steps
            return {"direction_weights": ((W0 - W) / scale, WA, float(n), None),
                    "direction_bias": ((b0 - b) / scale, WA, float(n), None),
                    "step_scale": (np.array([n * scale]), SUM, 1.0, None)}, None
        if self.name == "scaffold":
            inv = 1.0 / (steps * self.lr)
            cw = state["ctrl_weights"] - glob["server_ctrl_weights"][0] + (W0 - W) * inv
            cb = state["ctrl_bias"] - glob["server_ctrl_bias"][0] + (b0 - b) * inv
            res = {"delta_weights": (W - W0, WA, float(n), None),
                   "delta_bias": (b - b0, WA, float(n), None),
                   "ctrl_delta_weights": (cw - state["ctrl_weights"], SA, 1.0, None),
                   "ctrl_delta_bias": (cb - state["ctrl_bias"], SA, 1.0, None)}
            return res, {"ctrl_weights": cw, "ctrl_bias": cb}
        if self.name == "feddyn":
            hw = state["grad_corr_weights"] - self.alpha * (W - W0)
            hb = state["grad_corr_bias"] - self.alpha * (b - b0)
            return ({"weights": (W, SA, 1.0, None), "bias": (b, SA, 1.0, None)},
                    {"grad_corr_weights": hw, "grad_corr_bias": hb})
        raise ValueError(self.name)

    def server_rule(self, glob: dict, agg: dict, weights: dict) -> dict:
        """fedsim/trainer.py:232-234, :280-285, :340-348, :397-407."""
        out = {k: (v.copy(), op) for k, (v, op) in glob.items()}
        if self.name in ("fedavg", "fedprox"):
            out["weights"] = (agg["weights"].copy(), glob["weights"][1])
            out["bias"] = (agg["bias"].copy(), glob["bias"][1])
        elif self.name == "fednova":
            eff = float(agg["step_scale"][0]) / weights["direction_weights"]
            out["weights"] = (glob["weights"][0] - eff * agg["direction_weights"], WA)
            out["bias"] = (glob["bias"][0] - eff * agg["direction_bias"], WA)
        elif self.name == "scaffold":
            out["weights"] = (glob["weights"][0] + agg["delta_weights"], WA)
            out["bias"] = (glob["bias"][0] + agg["delta_bias"], WA)
            out["server_ctrl_weights"] = (glob["server_ctrl_weights"][0]
                                          + self.client_fraction * agg["ctrl_delta_weights"], SUM)
            out["server_ctrl_bias"] = (glob["server_ctrl_bias"][0]
                                       + self.client_fraction * agg["ctrl_delta_bias"], SUM)
        elif self.name == "feddyn":
            xw, xb = glob["weights"][0], glob["bias"][0]
            hw = glob["server_h_weights"][0] - self.alpha * self.client_fraction * (agg["weights"] - xw)
            hb = glob["server_h_bias"][0] - self.alpha * self.client_fraction * (agg["bias"] - xb)
            out["weights"] = (agg["weights"] - hw / self.alpha, SA)
            out["bias"] = (agg["bias"] - hb / self.alpha, SA)
            out["server_h_weights"] = (hw, SUM)
            out["server_h_bias"] = (hb, SUM)
        return out

    @property
    def required(self):
        """fedsim/trainer.py:183, :266, :300-301."""
        return {"fednova": ("direction_weights", "direction_bias", "step_scale"),
                "scaffold": ("delta_weights", "delta_bias",
                             "ctrl_delta_weights", "ctrl_delta_bias")}.get(
                                 self.name, ("weights", "bias"))


class NonFinite(RuntimeError):
    pass


def train_client(algo: Algo, X, y, client_id: int, glob: dict, state,
                 epochs: int, batch_size: int, lr: float, seed: int, rnd: int):
    """fedsim/trainer.py:427-477 (client_execute), minus wall-clock timing.

    Returns (result, new_state, steps, mean_loss)."""
    n = len(y)
    W0, b0 = glob["weights"][0], glob["bias"][0]
    bs = n if batch_size <= 0 else min(batch_size, n)
    W, b = W0.copy(), b0.copy()
    steps, loss_sum = 0, 0.0
    for order in minibatch_orders(seed, client_id, rnd, n, epochs):
        for lo in range(0, n, bs):
            idx = order[lo:lo + bs]
            loss, gW, gb = algo.gradient(W, b, X[idx], y[idx], W0, b0, glob, state)
            if not np.isfinite(loss):
                raise NonFinite(f"client {client_id} round {rnd}: loss diverged")
            W = W - lr * gW
            b = b - lr * gb
            loss_sum += loss
            steps += 1
    result, new_state = algo.finalize(W, b, steps, W0, b0, glob, state, n)
    if algo.collect_local_loss:
        result["local_loss"] = (np.array([loss_sum / steps]), COLLECT, 1.0, client_id)
    return result, new_state, steps, loss_sum / steps


# ---------------------------------------------------------------------------
# Hierarchical fold  (fedsim/aggregate.py:76-165)
# ---------------------------------------------------------------------------

def new_partial() -> dict:
    return {"entries": {}, "clients": []}


def fold_into(partial: dict, result: dict, client_id: int) -> dict:
    """fedsim/aggregate.py:76-102: WA acc += w*x, wsum += w; Sum/SA acc += x;
    Collect appends; count += 1; call order is fold order."""
    for name, (x, op, w, cid) in result.items():
        e = partial["entries"].setdefault(
            name, {"op": op, "acc": None, "wsum": 0.0, "count": 0, "items": []})
        if e["op"] != op:
            raise ValueError(f"op mismatch on {name}")
        if op == COLLECT:
            e["items"].append((cid, x))
        else:
            if e["acc"] is None:
                e["acc"] = np.zeros_like(x)
            if e["acc"].shape != x.shape:
                raise ValueError(f"shape mismatch on {name}")
            if op == WA:
                e["acc"] += w * x
                e["wsum"] += w
            else:
                e["acc"] += x
        e["count"] += 1
    partial["clients"].append(client_id)
    return partial


def combine(partials: list[dict]):
    """fedsim/aggregate.py:105-146: idle partials skipped, device-order sum,
    one divide.  Returns (tensors, collected, weights, counts, clients)."""
    live = [p for p in partials if p["entries"]]
    if not live:
        raise ValueError("no client results to aggregate")
    ops = {k: e["op"] for k, e in live[0]["entries"].items()}
    for p in live[1:]:
        if {k: e["op"] for k, e in p["entries"].items()} != ops:
            raise ValueError("schema mismatch")
    tensors, collected, weights, counts = {}, {}, {}, {}
    for name, op in ops.items():
        parts = [p["entries"][name] for p in live]
        counts[name] = sum(e["count"] for e in parts)
        if op == COLLECT:
            collected[name] = [it for e in parts for it in e["items"]]
            continue
        total = np.zeros_like(parts[0]["acc"])
        for e in parts:
            total += e["acc"]
        if op == WA:
            weights[name] = sum(e["wsum"] for e in parts)
            tensors[name] = total / weights[name]
        elif op == SA:
            tensors[name] = total / counts[name]
        else:
            tensors[name] = total
    clients = tuple(c for p in live for c in p["clients"])
    return tensors, collected, weights, counts, clients


# ---------------------------------------------------------------------------
# Scheduling  (fedsim/schedule.py:48-190) and device time model
# (fedsim/engine.py:427-450)
# ---------------------------------------------------------------------------

def greedy_plan(sizes: dict, selected, t, b):
    """fedsim/schedule.py:48-85,145-161: LPT order by (-N, id); each task goes to
    the device minimising (resulting makespan, resulting load, device id)."""
    order = sorted(selected, key=lambda m: (-sizes[m], m))
    k = len(t)
    load = [0.0] * k
    plan = {j: [] for j in range(k)}
    for m in order:
        hi = max(load)
        top = load.index(hi)
        rest = max([load[j] for j in range(k) if j != top], default=-np.inf)
        best = None
        for j in range(k):
            pred = float(sizes[m]) * float(t[j]) + float(b[j])
            pred = 0.0 if pred < 0.0 else pred
            cand = load[j] + pred
            other = rest if j == top else hi
            key = (max(cand, other), cand, j)
            if best is None or key < best:
                best = key
        plan[best[2]].append(int(m))
        load[best[2]] = best[1]
    return plan, load


def uniform_plan(selected, k: int) -> dict:
    """fedsim/schedule.py:135-142 (np.array_split semantics)."""
    n = len(selected)
    base, extra = divmod(n, k)
    out, pos = {}, 0
    for j in range(k):
        size = base + (1 if j < extra else 0)
        out[j] = [int(c) for c in selected[pos:pos + size]]
        pos += size
    return out


def ols_fit(samples, seconds):
    """fedsim/estimate.py:108-118."""
    n = np.asarray(samples, float)
    t = np.asarray(seconds, float)
    nc = n - n.mean()
    den = float(nc @ nc)
    if den == 0.0:
        return float(t.mean() / n.mean()), 0.0
    slope = float(nc @ (t - t.mean())) / den
    return slope, float(t.mean() - slope * n.mean())


# ---------------------------------------------------------------------------
# One SP round end to end  (fedsim/engine.py:748-812, SP branch)
# ---------------------------------------------------------------------------

def sp_round(algo: Algo, data, glob: dict, states: dict, seed: int, rnd: int,
             total: int, per_round: int, epochs: int):
    """Select, train every client in selection order on one device, fold,
    global fold, server rule.  ``data`` maps client -> (X, y); ``states`` maps
    client -> payload dict (mutated for stateful algorithms)."""
    sel = selection(seed, total, per_round, rnd)
    part = new_partial()
    for m in sel:
        X, y = data[m]
        st = None
        if algo.stateful:
            st = states.get(m) or algo.default_state(glob["weights"][0], glob["bias"][0])
        res, new_st, _, _ = train_client(algo, X, y, m, glob, st, epochs,
                                         algo.batch_size, algo.lr, seed, rnd)
        if new_st is not None:
            states[m] = new_st
        fold_into(part, res, m)
    tensors, _, weights, _, _ = combine([part])
    return algo.server_rule(glob, tensors, weights), sel
