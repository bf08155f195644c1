"""TEST INFRASTRUCTURE (never imported by the product path): numpy restatement
of the reference policy network's forward pass and action selection, the
checker for the device policy kernels (paper_2312_15122_b200/csrc/zsim_policy.cu).

Restates, from /root/reference/proj/src/core/:
  * nn/model.hpp:20-36    ModelConfig (latent 128, 2 heads, 2 trunk blocks,
                          value_embed 32, obs spec 16/128/64, 7 x 5 action bins)
  * nn/model.hpp:56-64    fixed input scales kActiveScale .. kValueScale
  * nn/model.hpp:101-167  ParamIndex::build -- flat parameter order, shapes
  * nn/model.hpp:199-212  Model::init -- uniform(+-1/sqrt(fan_in)) from Rng(seed)
  * nn/model.hpp:287-303  ln_forward (eps 1e-5, biased variance)
  * nn/model.hpp:326-367  attn_forward (pre-LN MHA, masked keys get p = 0)
  * nn/model.hpp:431-440  mlp_forward (pre-LN, GELU(erf), residual)
  * nn/model.hpp:464-585  forward_row
  * nn/model.hpp:672-705  log_softmax, sample_categorical, argmax
  * train/policy.hpp:27-58 NNPolicy::act
  * common.hpp:28-44       Rng (splitmix64)

Parity pinning: the reference model is Eigen code and Eigen is absent from
this image, so the reference forward pass cannot be built or run here --
parity of the forward pass is UNPINNED (this restatement is the checker).
The parameter layout and Model::init ARE pinned: they depend only on Rng,
whose restatement is pinned bit-exact by the simulator oracle, and
tests/test_policy.py checks the device library's init against this file
bit for bit.  Arithmetic here is float64 throughout (the reference computes
in float32 with Eigen's summation order), so the oracle is the "exact"
value both sides are compared against with a stated tolerance.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1

ACTIVE_SCALE = np.array([0.1, 1.8, 0.02, 1, 1, 1, 1, 0.02, 0.1], np.float32)   # model.hpp:56-57
AGENT_SCALE = np.array([0.02, 0.02, 0.32, 0.1, 0.02, 1], np.float32)           # model.hpp:58-59
ROAD_SCALE = np.array([0.02, 0.02] + [1] * 10, np.float32)                     # model.hpp:60-61
ROUTE_SCALE = np.array([0.02, 0.02, 1, 1, 1], np.float32)                      # model.hpp:62
VALUE_SCALE = np.array([0.02, 0.01], np.float32)                               # model.hpp:63
AGENT_F, ROAD_F, ROUTE_F, ACTIVE_F, VALUE_F = 6, 12, 5, 9, 2                   # simcore.hpp:65-69
LN_EPS = 1e-5                                                                  # model.hpp:285


@dataclass
class ModelConfig:
    """nn/model.hpp:20-36."""
    latent: int = 128
    heads: int = 2
    trunk_blocks: int = 2
    value_embed: int = 32
    n_agents: int = 16
    n_road: int = 128
    n_route: int = 64
    n_accel: int = 7
    n_steer: int = 5


class Rng:
    """common.hpp:28-44 (splitmix64)."""

    def __init__(self, seed: int = 0, state: int | None = None):
        self.state = (seed + 0x9E3779B97F4A7C15) & M64 if state is None else state

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53


@dataclass
class Entry:
    name: str
    offset: int
    rows: int
    cols: int
    is_weight: bool
    init: float


@dataclass
class ParamIndex:
    entries: list = field(default_factory=list)
    total: int = 0
    by_name: dict = field(default_factory=dict)

    def add(self, name, rows, cols, is_weight, init=0.0):
        e = Entry(name, self.total, rows, cols, is_weight, init)
        self.entries.append(e)
        self.by_name[name] = e
        self.total += rows * cols
        return e


def param_index(cfg: ModelConfig) -> ParamIndex:
    """ParamIndex::build (model.hpp:101-167): same names, order and shapes."""
    ix = ParamIndex()
    d = cfg.latent

    def attn(p):
        ix.add(p + ".ln.g", d, 1, False, 1.0)
        ix.add(p + ".ln.b", d, 1, False, 0.0)
        for w in "qkvo":
            ix.add(f"{p}.w{w}", d, d, True)
            ix.add(f"{p}.b{w}", d, 1, False)

    def block(p, width):
        ix.add(p + ".ln.g", width, 1, False, 1.0)
        ix.add(p + ".ln.b", width, 1, False, 0.0)
        ix.add(p + ".w1", width, width, True)
        ix.add(p + ".b1", width, 1, False)
        ix.add(p + ".w2", width, width, True)
        ix.add(p + ".b2", width, 1, False)

    ix.add("emb.agents.w", d, AGENT_F, True)
    ix.add("emb.agents.b", d, 1, False)
    ix.add("emb.road.w", d, ROAD_F, True)
    ix.add("emb.road.b", d, 1, False)
    ix.add("emb.route.w", d, ROUTE_F, True)
    ix.add("emb.route.b", d, 1, False)
    ix.add("emb.active.w", d, ACTIVE_F, True)
    ix.add("emb.active.b", d, 1, False)
    for n in ("agents", "road", "route", "active"):
        ix.add("null." + n, d, 1, True)
    attn("enc.self")
    attn("enc.cross.road")
    attn("enc.cross.route")
    attn("enc.cross.active")
    for i in range(cfg.trunk_blocks):
        block(f"policy.block{i}", d)
    ix.add("policy.accel.w", cfg.n_accel, d, True)
    ix.add("policy.accel.b", cfg.n_accel, 1, False)
    ix.add("policy.steer.w", cfg.n_steer, d, True)
    ix.add("policy.steer.b", cfg.n_steer, 1, False)
    ix.add("value.emb.w", cfg.value_embed, VALUE_F, True)
    ix.add("value.emb.b", cfg.value_embed, 1, False)
    ix.add("value.in.w", d, d + cfg.value_embed, True)
    ix.add("value.in.b", d, 1, False)
    for i in range(cfg.trunk_blocks):
        block(f"value.block{i}", d)
    ix.add("value.head.w", 1, d, True)
    ix.add("value.head.b", 1, 1, False)
    return ix


def init_params(cfg: ModelConfig, seed: int) -> np.ndarray:
    """Model::init (model.hpp:199-212): float(lo + (hi - lo) * u) per element
    in flat order; fan_in = cols (rows for column vectors)."""
    ix = param_index(cfg)
    out = np.zeros(ix.total, np.float32)
    rng = Rng(seed)
    for e in ix.entries:
        n = e.rows * e.cols
        if e.is_weight:
            bound = 1.0 / math.sqrt(float(e.rows if e.cols == 1 else e.cols))
            lo, hi = -bound, bound
            out[e.offset:e.offset + n] = [lo + (hi - lo) * rng.uniform() for _ in range(n)]
        else:
            out[e.offset:e.offset + n] = e.init
    return out


class Model:
    """Model<T> with column-major Eigen maps (model.hpp:183-197), in float64."""

    def __init__(self, cfg: ModelConfig, params: np.ndarray):
        self.cfg = cfg
        self.ix = param_index(cfg)
        assert params.size == self.ix.total
        self.p = params.astype(np.float64)

    def mat(self, name):
        e = self.ix.by_name[name]
        return self.p[e.offset:e.offset + e.rows * e.cols].reshape(e.cols, e.rows).T  # column-major

    def vec(self, name):
        e = self.ix.by_name[name]
        return self.p[e.offset:e.offset + e.rows * e.cols]


def _ln(m, p, x):
    """ln_forward over the columns of x [d, n] (model.hpp:287-303)."""
    mu = x.mean(axis=0)
    var = ((x - mu) ** 2).sum(axis=0) / x.shape[0]
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    return (x - mu) * rstd * m.vec(p + ".ln.g")[:, None] + m.vec(p + ".ln.b")[:, None]


def _attn(m, p, x, kv, mask, self_mode):
    """attn_forward (model.hpp:326-367)."""
    d, heads = m.cfg.latent, m.cfg.heads
    dh = d // heads
    ln = _ln(m, p, x)
    src = ln if self_mode else kv
    q = m.mat(p + ".wq") @ ln + m.vec(p + ".bq")[:, None]
    k = m.mat(p + ".wk") @ src + m.vec(p + ".bk")[:, None]
    v = m.mat(p + ".wv") @ src + m.vec(p + ".bv")[:, None]
    scale = 1.0 / math.sqrt(dh)
    concat = np.zeros_like(q)
    msk = np.asarray(mask, bool)
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        s = (q[sl].T @ k[sl]) * scale
        s[:, ~msk] = -1e30
        pr = np.exp(s - s.max(axis=1, keepdims=True))
        pr /= pr.sum(axis=1, keepdims=True)
        concat[sl] = v[sl] @ pr.T
    return m.mat(p + ".wo") @ concat + m.vec(p + ".bo")[:, None] + x


def _gelu(x):
    return 0.5 * x * (1.0 + np.vectorize(math.erf)(x * 0.70710678118654752440))


def _mlp(m, p, x):
    """mlp_forward (model.hpp:431-440) on a vector."""
    ln = _ln(m, p, x[:, None])[:, 0]
    h = _gelu(m.mat(p + ".w1") @ ln + m.vec(p + ".b1"))
    return m.mat(p + ".w2") @ h + m.vec(p + ".b2") + x


def forward_row(m: Model, obs: dict, b: int):
    """forward_row (model.hpp:464-585) for row b of an observation batch given
    as numpy arrays {active [B,9], agents [B,Ka,6], road [B,Kr,12],
    route [B,Kl,5], value_only [B,2]}.  Returns (logits_accel, logits_steer,
    value) in float64."""
    ag = np.asarray(obs["agents"][b], np.float32)
    rd = np.asarray(obs["road"][b], np.float32)
    rt = np.asarray(obs["route"][b], np.float32)
    ac = np.asarray(obs["active"][b], np.float32)
    vf = np.asarray(obs["value_only"][b], np.float32)
    f_ag = (ag.astype(np.float64) * AGENT_SCALE.astype(np.float64)).T     # [6, na]
    f_rd = (rd.astype(np.float64) * ROAD_SCALE.astype(np.float64)).T
    f_rt = (rt.astype(np.float64) * ROUTE_SCALE.astype(np.float64)).T
    f_ac = (ac.astype(np.float64) * ACTIVE_SCALE.astype(np.float64))[:, None]
    f_v = vf.astype(np.float64) * VALUE_SCALE.astype(np.float64)

    mask_lat = np.concatenate([[True], ag[:, 5] > 0.5])
    x0 = np.concatenate([m.vec("null.agents")[:, None],
                         m.mat("emb.agents.w") @ f_ag + m.vec("emb.agents.b")[:, None]], axis=1)

    def kv(name, feats, raw, valid_at):
        t = np.concatenate([m.vec("null." + name)[:, None],
                            m.mat(f"emb.{name}.w") @ feats + m.vec(f"emb.{name}.b")[:, None]], axis=1)
        msk = np.concatenate([[True], (raw[:, valid_at] > 0.5) if valid_at >= 0 else np.ones(raw.shape[0], bool)])
        return t, msk

    x1 = _attn(m, "enc.self", x0, x0, mask_lat, True)
    t, k = kv("road", f_rd, rd, 11)
    x2 = _attn(m, "enc.cross.road", x1, t, k, False)
    t, k = kv("route", f_rt, rt, 4)
    x3 = _attn(m, "enc.cross.route", x2, t, k, False)
    t, k = kv("active", f_ac, ac[None, :], -1)
    x4 = _attn(m, "enc.cross.active", x3, t, k, False)
    pooled = x4[:, mask_lat].sum(axis=1) / mask_lat.sum()

    h = pooled
    for i in range(m.cfg.trunk_blocks):
        h = _mlp(m, f"policy.block{i}", h)
    la = m.mat("policy.accel.w") @ h + m.vec("policy.accel.b")
    ls = m.mat("policy.steer.w") @ h + m.vec("policy.steer.b")
    ve = _gelu(m.mat("value.emb.w") @ f_v + m.vec("value.emb.b"))
    hv = m.mat("value.in.w") @ np.concatenate([pooled, ve]) + m.vec("value.in.b")
    for i in range(m.cfg.trunk_blocks):
        hv = _mlp(m, f"value.block{i}", hv)
    value = float((m.mat("value.head.w") @ hv)[0] + m.vec("value.head.b")[0])
    return la, ls, value


def log_softmax(z):
    """model.hpp:672-678."""
    s = z - z.max()
    return s - math.log(np.exp(s).sum())


def argmax(z) -> int:
    """model.hpp:699-705: first maximum."""
    best = 0
    for i in range(1, len(z)):
        if z[i] > z[best]:
            best = i
    return best


def sample_categorical(z, rng: Rng):
    """model.hpp:680-697: inverse CDF over exp(log_softmax) with u = rng.uniform()."""
    ls = log_softmax(z)
    u = rng.uniform()
    acc, pick = 0.0, len(ls) - 1
    for i in range(len(ls)):
        acc += math.exp(ls[i])
        if u < acc:
            pick = i
            break
    return pick, float(ls[pick]), u


def act(m: Model, obs: dict, rng_state: np.ndarray, use_argmax: bool):
    """NNPolicy::act (policy.hpp:27-58) over every row: returns accel, steer,
    logp, value, the advanced rng states and the raw logits."""
    B = len(obs["active"])
    out = dict(accel=np.zeros(B, np.int32), steer=np.zeros(B, np.int32), logp=np.zeros(B),
               value=np.zeros(B), rng=np.array(rng_state, np.uint64).copy(),
               logits_accel=np.zeros((B, m.cfg.n_accel)), logits_steer=np.zeros((B, m.cfg.n_steer)),
               u=np.zeros((B, 2)))
    for b in range(B):
        la, ls, v = forward_row(m, obs, b)
        out["logits_accel"][b], out["logits_steer"][b], out["value"][b] = la, ls, v
        if use_argmax:
            ai, si = argmax(la), argmax(ls)
            out["logp"][b] = log_softmax(la)[ai] + log_softmax(ls)[si]
        else:
            r = Rng(state=int(out["rng"][b]))
            ai, lpa, ua = sample_categorical(la, r)
            si, lps, us = sample_categorical(ls, r)
            out["logp"][b] = lpa + lps
            out["rng"][b] = np.uint64(r.state)
            out["u"][b] = (ua, us)
        out["accel"][b], out["steer"][b] = ai, si
    return out
