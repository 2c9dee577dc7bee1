"""Instruction mix of the hottest (innermost, largest) loop of a kernel's SASS (dev aid).

    python tools/sass_loop.py <obj or .so> <kernel-name regex>
Prints, per matching kernel, the opcode histogram of every backward-branch loop body of >= 64
instructions that contains an mbarrier wait or a barrier (the per-plane / per-row loops)."""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], re.compile(sys.argv[2])
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs, cur = {}, None
for ln in out.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
for f, ins in funcs.items():
    if not pat.search(f):
        continue
    loops = []
    for a, t in ins:
        m = re.search(r"\bBRA(?:\.\S+)?\s+(?:\S+,\s*)?(?:`\()?.*?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) <= a:
            body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
            if len(body) >= 64:
                loops.append((int(m.group(1), 16), a, body))
    print(f"== {f}  ({len(ins)} instructions)")
    for lo, hi, body in sorted(loops, key=lambda l: l[1] - l[0])[:3]:
        ops = collections.Counter()
        for _, t in body:
            t = re.sub(r"^@!?U?P\w+\s+", "", t)
            ops[t.split()[0].split(".")[0]] += 1
        print(f"  loop {lo:#x}-{hi:#x}: {len(body)} instr: " +
              ", ".join(f"{k} {v}" for k, v in ops.most_common(18)))
