"""Dev helper: print one kernel's SASS from a .so (cuobjdump), optionally only a loop."""
import re, subprocess, sys
so, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if re.search(pat, name):
        print("Function:", name)
        for line in f.split("\n")[1:]:
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                print(m.group(1), m.group(2).strip())
        break
