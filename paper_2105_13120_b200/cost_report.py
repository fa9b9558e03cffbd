"""Communication reconciliation: the reference's cost model against what this package's
rings charge and actually send.

The reference's analytic communication volumes (ringseq/cost_model.py:122-168) are
restated here in exact ``Fraction`` arithmetic:

* ``_collective_unit`` (:122-127): 2(N-1)*B*Z*(L/N)*A elements per device, the cost of one
  K or V circulation pair in the ring and of one (B, L, H) all-reduce;
* ``comm_volume`` (:130-150), sequence scheme: forward = unit, backward = 3 * unit per
  attention block (the MLP block communicates nothing);
* ``sparse_comm_volume`` (:153-159): (N-1)*2*B*Z*K*A for the Linformer's two partial
  circulations.

``reconcile`` puts three things side by side for one configuration:

1. the model's element counts;
2. the ledger element counts the API returns (``forward_ledger`` / ``backward_ledger``:
   the reference's charging convention, ringseq/cluster.py:130-135), which must equal (1)
   exactly;
3. the bytes each transport plan puts on the wire per device and layer: the paper's
   plan (bf16 K/V rings, fp32 partial all-reduces), this package's panel mode (one K/V
   pair ring forward, cached K/V, fp32 reduce-scatter), and its stream mode (the K/V pair
   ring twice plus N hops of the fp32 dK/dV sums).  With ``measured`` (a ledger's
   ``wire_bytes`` per device from a real ``SpmdRing`` run) the measured bytes are checked
   against the plan.  Link time at 900 GB/s per direction (NVLink 5) is reported next to
   each.
"""

from __future__ import annotations

from fractions import Fraction

from .config import AttentionConfig, SparseAttentionConfig

__all__ = ["collective_unit", "comm_volume", "sparse_comm_volume", "wire_bytes", "reconcile"]

NVLINK_BYTES_PER_S = 900e9


def collective_unit(cfg: AttentionConfig) -> Fraction:
    """2(N-1)*B*Z*(L/N)*A elements (ringseq/cost_model.py:122-127)."""
    n = cfg.num_devices
    return Fraction(2 * (n - 1) * cfg.batch_size * cfg.num_heads * cfg.seq_len * cfg.head_size, n)


def comm_volume(cfg: AttentionConfig, direction: str = "total") -> Fraction:
    """Sequence-scheme attention elements per device and layer (ringseq/cost_model.py:130-150)."""
    unit = collective_unit(cfg)
    per = {"forward": unit, "backward": 3 * unit}
    if direction == "total":
        return per["forward"] + per["backward"]
    return per[direction]


def sparse_comm_volume(cfg: SparseAttentionConfig) -> Fraction:
    """(N-1)*2*B*Z*K*A elements per device (ringseq/cost_model.py:153-159)."""
    b = cfg.base
    return Fraction((b.num_devices - 1) * 2 * b.batch_size * b.num_heads * cfg.proj_dim * b.head_size)


def wire_bytes(cfg: AttentionConfig, plan: str, kv_bytes: int = 2, grad_bytes: int = 4) -> dict:
    """Bytes one device sends per layer (forward, backward) under a transport plan."""
    n = cfg.num_devices
    chunk = cfg.batch_size * cfg.num_heads * cfg.chunk_len * cfg.head_size  # C elements
    full = n * chunk
    ring = 2 * (n - 1) * chunk  # one K and one V circulation (or one K/V pair ring)
    if n == 1:
        return {"forward": 0, "backward": 0}
    if plan == "paper":  # bf16 rings; two fp32 all-reduces of (B, Z, L, A), ring all-reduce bytes
        return {"forward": ring * kv_bytes,
                "backward": ring * kv_bytes + 2 * (2 * (n - 1) * full * grad_bytes // n)}
    if plan == "panel":  # K/V cached by the forward: no backward ring; reduce-scatter of the partials
        return {"forward": ring * kv_bytes, "backward": 2 * ((n - 1) * full * grad_bytes // n)}
    if plan == "panel_paper":  # cached K/V, all-reduce of the partials (mode="paper")
        return {"forward": ring * kv_bytes, "backward": 2 * (2 * (n - 1) * full * grad_bytes // n)}
    if plan == "stream":  # the pair ring again, plus N hops of the two fp32 sums
        return {"forward": ring * kv_bytes, "backward": ring * kv_bytes + 2 * n * chunk * grad_bytes}
    raise ValueError(f"unknown plan {plan!r}")


def reconcile(cfg: AttentionConfig, sparse: SparseAttentionConfig | None = None, measured: dict | None = None,
              plan: str = "panel") -> dict:
    """Model vs ledger vs wire bytes for one configuration (see the module docstring).

    ``measured``: {"forward": bytes, "backward": bytes} one device actually sent (e.g. the
    difference of ``SpmdRing.ledger.devices[d].wire_bytes`` around a layer's forward and
    backward) under ``plan``."""
    from .ring_attention import backward_ledger, forward_ledger

    fl, bl = forward_ledger(cfg), backward_ledger(cfg)
    ledger = {
        "forward": max(Fraction(t.ring_p2p_elements) + Fraction(t.allreduce_elements) for t in fl.devices),
        "backward": max(Fraction(t.ring_p2p_elements) + Fraction(t.allreduce_elements) for t in bl.devices),
    }
    model = {"forward": comm_volume(cfg, "forward"), "backward": comm_volume(cfg, "backward")}
    out = {
        "config": {"B": cfg.batch_size, "Z": cfg.num_heads, "L": cfg.seq_len, "A": cfg.head_size,
                   "N": cfg.num_devices},
        "model_elements": {k: str(v) for k, v in model.items()},
        "ledger_elements": {k: str(v) for k, v in ledger.items()},
        "ledger_matches_model": all(ledger[k] == model[k] for k in model),
        "plans": {},
    }
    for p in ("paper", "panel", "panel_paper", "stream"):
        wb = wire_bytes(cfg, p)
        out["plans"][p] = {**wb, "total": wb["forward"] + wb["backward"],
                           "link_us": (wb["forward"] + wb["backward"]) / NVLINK_BYTES_PER_S * 1e6}
    if measured is not None:
        want = wire_bytes(cfg, plan)
        out["measured"] = {"plan": plan, **measured,
                           "matches_plan": all(int(measured[k]) == int(want[k]) for k in ("forward", "backward"))}
    if sparse is not None:
        from .cluster import CommLedger  # noqa: F401  (ledger convention: ring-accumulate)

        out["sparse_model_elements"] = str(sparse_comm_volume(sparse))
        base = sparse.base
        out["sparse_wire_bytes_allreduce"] = (2 * (base.num_devices - 1) * 2 * base.batch_size * base.num_heads
                                              * sparse.proj_dim * base.head_size * 4 // base.num_devices)
    return out
