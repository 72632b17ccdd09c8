"""Registers / spills per kernel instantiation from the build's ptxas logs (lib/ptxas_*.log).
usage: python tools/ptxas_summary.py qed_eval_N4 [qed_regs_N2 ...]"""
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2511_19456_b200", "lib")
for tag in sys.argv[1:]:
    txt = open(os.path.join(LIB, f"ptxas_{tag}.log")).read()
    rows = re.findall(r"Compiling entry function '(\S+)'.*?(\d+) bytes spill stores.*?Used (\d+) registers", txt, re.S)
    names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
    for (m, sp, rg), nm in zip(rows, names):
        nm = re.sub(r"qed::|qedgen_N\d+(_p\d+)?::|qedregs_N\d+::|qedbg_N\d+::|\(qed::QedEvalArgs\)|\(qed::QedMcArgs\)", "", nm)
        print(f"{tag:14s} regs {rg:>3s} spill {sp:>4s}  {nm}")
