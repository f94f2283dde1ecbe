"""Prints DESIGN.md §6's result tables from the committed bench lines and
predicted-vs-measured files (profiles/round1_final_n{1,2,4}_*.json,
profiles/round1_predict_vs_measured_n{2,4}_*.json). No GPU."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"gpt2-1.3b-dp": "GPT-2 1.3B DP (2)", "llama3-8b-tp-sp": "Llama-3 8B TP-SP (3)",
         "llama3-70b-fsdp": "Llama-3 70B-layer FSDP (4)", "mixtral-8x7b-ep": "Mixtral 8x7B EP (5)"}


def prof(name):
    return json.load(open(os.path.join(ROOT, "profiles", name)))


def bench_rows():
    out = ["| workload (BASELINE config) | N | Lagom-tuned | NCCL-default | speedup | Lagom picks | "
           "compute slowdown (Lagom / NCCL) | roofline frac |", "|---|---|---|---|---|---|---|---|"]
    for n in (4, 2):
        for w, name in NAMES.items():
            l = prof(f"round1_final_n{n}_{w}.json")["line"]
            c = l["compute"]
            ncs = sorted({int(p.split("/NC")[1].split("/")[0]) for p in l["config"]["tune"]["picks"]})
            nc = f"NC{ncs[0]}" if len(ncs) == 1 else f"NC{ncs[0]}–{ncs[-1]}"
            kind = "A2A one-hop" if w.startswith("mixtral") else "NVLS"
            sp = l["speedup_vs_nccl_default"]
            sps = f"**{sp:.3f}×**" if sp >= 1.07 else f"{sp:.3f}×"
            out.append(f"| {name} | {n} | {l['value']:.2f} | {l['nccl_default_ms']:.2f} | {sps} | TREE ({kind}) {nc} | "
                       f"{c['slowdown']:.3f} / {c['slowdown_nccl']:.3f} | {l['roofline']['frac']:.3f} |")
    l = prof("round1_final_n1_gpt2-1.3b-dp.json")["line"]
    c = l["compute"]
    out.append(f"| GPT-2 1.3B DP (2) | 1 | {l['value']:.2f} | {l['nccl_default_ms']:.2f} | "
               f"{l['speedup_vs_nccl_default']:.3f}× | copy NC8/NT512 | {c['slowdown']:.3f} / {c['slowdown_nccl']:.3f} | "
               f"{l['roofline']['frac']:.3f} (HBM; 8 of 148 SMs) |")
    return "\n".join(out)


def pvm_rows():
    out = ["| workload | N | predicted Z (ms) | measured Z (ms) | Z error | Y error | X error |",
           "|---|---|---|---|---|---|---|"]
    for n in (4, 2):
        for w, name in NAMES.items():
            p = prof(f"round1_predict_vs_measured_n{n}_{w}.json")
            e = p["rel_err"]
            out.append(f"| {name} | {n} | {p['predicted']['Z'] / 1e3:.2f} | {p['measured']['Z'] / 1e3:.2f} | "
                       f"{e['Z'] * 100:+.1f} % | {e['Y'] * 100:+.1f} % | {e['X'] * 100:+.1f} % |")
    return "\n".join(out)


if __name__ == "__main__":
    print(bench_rows())
    print()
    print(pvm_rows())
