"""Communication reconciliation for BASELINE.json's configs (paper_2105_13120_b200.cost_report):
the reference's model (ringseq/cost_model.py:122-159) vs the ledgers vs each transport plan's bytes.

usage: python tools/comm_report.py [--out profiles/r2_comm_report.json]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import AttentionConfig, SparseAttentionConfig  # noqa: E402
from paper_2105_13120_b200.cost_report import reconcile  # noqa: E402


def cfg(b, z, seq, a, n):
    return AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)


CONFIGS = {
    "config1_N4": cfg(4, 12, 512, 64, 4),
    **{f"config2_N{n}": cfg(64 * n, 12, 512, 64, n) for n in (2, 4, 8)},
    "config3_L16K_N8": cfg(4, 12, 16384, 64, 8),
    "config4_N8": cfg(4, 16, 16384, 64, 8),
}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r2_comm_report.json")
    args = ap.parse_args()
    rep = {k: reconcile(c) for k, c in CONFIGS.items()}
    rep["config5_linformer_N8"] = reconcile(cfg(4, 12, 114688, 64, 8),
                                            sparse=SparseAttentionConfig(base=cfg(4, 12, 114688, 64, 8), proj_dim=256))
    Path(args.out).write_text(json.dumps(rep, indent=1))
    for k, r in rep.items():
        p = r["plans"]
        print(f"{k:22s} ledger==model {r['ledger_matches_model']}  link us/layer: paper {p['paper']['link_us']:.0f}, "
              f"panel {p['panel']['link_us']:.0f}, stream {p['stream']['link_us']:.0f}")
