import re, sys
txt = open(sys.argv[1]).read().splitlines()
cur = None
for line in txt:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1); continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur2 = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur: stack = m.groups(); continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = re.sub(r"_ZN3cpb\d+_GLOBAL__N__\w+?_\d+_cpb_\w+?_cu_\w+?\d+", "", cur)[:60]
        print(f"{name:60s} regs={m.group(1):>4} stack/spill={stack}")
        cur = None
