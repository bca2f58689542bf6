"""Print the scoreboard control fields (write/read barrier set, wait mask, stall) of a kernel's SASS, optionally
only for one address range: shows whether shared-memory lookups share a scoreboard with global loads.

    python scripts/sass_sb.py LIB.so KERNEL_REGEX [START_HEX END_HEX]
"""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
lo, hi = (int(sys.argv[3], 16), int(sys.argv[4], 16)) if len(sys.argv) > 4 else (0, 1 << 40)
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out):
    name = f.split("\n")[0]
    if not re.search(pat, name):
        continue
    print(name)
    lines = f.split("\n")
    for i, l in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", l)
        if not m or i + 1 >= len(lines):
            continue
        m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        a = int(m.group(1), 16)
        if not (lo <= a <= hi) or not m2:
            continue
        c = int(m2.group(1), 16) >> 41
        stall, wb, rb, wait = c & 0xF, (c >> 5) & 7, (c >> 8) & 7, (c >> 11) & 0x3F
        print(f"{a:05x} {m.group(2)[:60]:60s} st={stall:2d} wb={wb if wb != 7 else '-'} rb={rb if rb != 7 else '-'} "
              f"wait={wait:06b}")
    break
