"""Static check of the tile engine's code generation: instruction mix of every DMMA-dense loop body of a kernel
(the 32-deep k slice of the update tile is 256 DMMA; ~1660 instructions is the good schedule, ~1830 the bad one).
    python tools/sass_loopstat.py paper_1611_06365_b200/libmla_b200.so _Z7k_getrfN3mla9GetrfArgsE [max_body]
"""
import sys, re, subprocess
lib, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout.splitlines()
start = [i for i, l in enumerate(out) if "Function :" in l]
names = {out[i].split("Function :")[1].strip(): i for i in start}
i0 = names[fn]; i1 = min([i for i in start if i > i0] + [len(out)])
ins = []
for l in out[i0:i1]:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
# find backward branches enclosing DMMA-dense regions
addr_idx = {a: k for k, (a, _) in enumerate(ins)}
loops = []
for k, (a, t) in enumerate(ins):
    m = re.search(r"BRA\S*\s+(?:\S+,\s*)?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr_idx:
            body = ins[addr_idx[tgt]:k + 1]
            nd = sum(1 for _, x in body if "DMMA" in x)
            if nd >= 128 and len(body) <= (int(sys.argv[3]) if len(sys.argv) > 3 else 4000):
                loops.append((tgt, a, body, nd))
for tgt, a, body, nd in loops:
    ops = {}
    for _, x in body:
        op = x.split()[0] if not x.startswith("@") else x.split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = sorted(ops.items(), key=lambda kv: -kv[1])[:12]
    local = sum(v for k, v in ops.items() if k in ("LDL", "STL"))
    print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr, DMMA {nd}, local-memory ops {local}, R2UR {ops.get('R2UR', 0)} | " + " ".join(f"{k}:{v}" for k, v in top))
