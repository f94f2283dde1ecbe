#!/usr/bin/env python3
"""Regenerates the committed golden fixtures from the REFERENCE build
(oracle/_ref/parity_driver_ref = tests/cpp/parity_driver.cpp compiled against
/root/reference/proj/src with -Dlagom=lagom_ref -ffp-contract=off; recipe in
oracle/Makefile). Needs /root/reference, i.e. runs in the build container.

Outputs (tests/golden/):
  parity_ref.digests   one line per driver case: "<case> <sha256 of its JSON line>"
                       (1858 cases: generators, simulate, tune in both start
                       modes incl. the 600 SURVEY-A.4 runs, scripted profile
                       tables, oracles, sweeps, cost model, JSON I/O, errors)
  parity_ref_key.jsonl the full JSON lines of the human-readable key cases
                       (allreduce-pair tune logs, model table, A.3 variants)
"""
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
KEY = ("tune/allreduce_pair/min/b500", "tune/allreduce_pair/nccl/b500", "tune/variant_cb/min",
       "tune/variant_bal/min", "model/RING/SIMPLE/P2P", "model/select_subspace", "model/params_json",
       "oracle/allreduce_pair", "naive/allreduce_pair", "sweep/0")


def main():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "parity_driver_ref")], check=True,
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    with open(os.path.join(HERE, "parity_ref.digests"), "w") as f:
        for ln in lines:
            case = ln[len('{"case":"'):].split('"', 1)[0]
            f.write(f"{case} {hashlib.sha256(ln.encode()).hexdigest()}\n")
    with open(os.path.join(HERE, "parity_ref_key.jsonl"), "w") as f:
        for ln in lines:
            case = ln[len('{"case":"'):].split('"', 1)[0]
            if case in KEY:
                f.write(ln + "\n")
    print(f"{len(lines)} cases written", file=sys.stderr)


if __name__ == "__main__":
    main()
