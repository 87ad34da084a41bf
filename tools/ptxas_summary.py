"""Summarise `nvcc -Xptxas -v` output: kernel, registers, stack, spills."""
import re, sys
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"(k_[a-z0-9_]+)(I[LiE0-9]+E)?", name)
        cur = (k.group(1) + (re.sub(r"[LiE]", " ", k.group(2)).split().__str__() if k.group(2) else "")) if k else name
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        stack = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:45s} regs={m.group(1):>4s} stack={stack[0]} spill_st={stack[1]} spill_ld={stack[2]}")
        cur = None
