"""Static SASS instruction count per source-line range of a kernel (nvdisasm -gi):
python tools/sass_lines.py file.cubin kernel_substring file.cu lo-hi[:name] ..."""
import re
import subprocess
import sys

cubin, kern, src = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    span, _, name = a.partition(":")
    lo, hi = map(int, span.split("-"))
    ranges.append((lo, hi, name or span))
out = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
cur_fn, line, counts, total, prev_marker = None, None, {}, 0, False
for l in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur_fn = m.group(1)
        continue
    if cur_fn is None or kern not in cur_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if not prev_marker:  # the innermost location comes first in a group of markers
            line = (m.group(1).split("/")[-1], int(m.group(2)))
        prev_marker = True
        continue
    prev_marker = False
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        total += 1
        if line:
            counts[line] = counts.get(line, 0) + 1
print("total SASS", total)
for lo, hi, name in ranges:
    print(f"{name:<20} {sum(v for (f, ln), v in counts.items() if f == src and lo <= ln <= hi)}")
