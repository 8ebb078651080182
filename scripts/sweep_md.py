"""Render a scripts/sweep.py JSONL file as the markdown table of profiles/rNN_sweep.md.
    python scripts/sweep_md.py <sweep.jsonl> <title>"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print(f"# {sys.argv[2]}\n")
print("One B200, Infinity-1K schedule, 1 x 16 heads (2B shape), D=128, bf16, `structured` synthetic "
      "inputs (seed 0, DESIGN.md §4).  ms = median CUDA-event time of one attention launch over all 16 "
      "heads; util = executed FLOPs / (ms x measured burst bf16 peak); error = block-sparse output vs "
      "the build's own dense kernel (relative Frobenius / max abs) — the method error of the pattern on "
      "these synthetic inputs, not a kernel error.  CS4A points use the paper's sink order (READING 25).\n")
for B in sorted({r["B"] for r in rows}, reverse=True):
    print(f"## B = {B}\n")
    print("| kind | K | setting | sink | blocks/head | FlexAttn sparsity | ms | dense ms | x dense | util | rel-F err | max err |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        if r["B"] != B:
            continue
        if "windows_11_12_13" in r:
            setting = "windows 11/12/13 = " + "/".join(str(x) for x in r["windows_11_12_13"])
        elif "windows_rel" in r:
            setting = "windows (rel) " + "/".join(str(x) for x in r["windows_rel"])
        else:
            setting = f"S={r['decision_scale']} {r['select']} {r['value']}"
        sink = r.get("sink_scales", 5)
        print(f"| {r['kind']} | {r['K']} | {setting} | {sink if sink else 'none'} | "
              f"{r['active_blocks_per_head']:.1f} | {100 * r['flex_sparsity']:.2f}% | {r['ms']:.4f} | "
              f"{r['dense_ms']:.4f} | {r['speedup_vs_dense']:.2f} | {100 * r['tensor_util_executed']:.1f}% | "
              f"{r['err_rel_fro_vs_dense']:.3f} | {r['err_max_abs_vs_dense']:.3f} |")
    print()
