"""Summarise build/ptxas.log: kernel, registers, stack, spill bytes (build-time check)."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "build/ptxas.log").read().splitlines()
name = None
for i, line in enumerate(log):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        name = re.sub(r"^_ZN5fvsrn\d+", "", name)
        name = re.sub(r"EEEv.*", ">", name).replace("ILi", "<").replace("ELi", ",").replace("ELin", ",-")
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        stack, st, ld = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if len(sys.argv) < 3 or re.search(sys.argv[2], name):
            print(f"{name:45s} regs={m.group(1):>4} stack={stack:>4} spill_st={st:>4} spill_ld={ld:>4}")
        name = None
