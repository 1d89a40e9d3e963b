"""TEST INFRASTRUCTURE: copy the C++ shim documented in INTEGRATION.md (its
first ```cpp block) verbatim into oracle/_ref/integration_shim.inc, so the
drop-in check compiles exactly the code a maintainer would paste."""
import os
import re
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
text = open(os.path.join(root, "INTEGRATION.md")).read()
code = re.search(r"```cpp\n(.*?)```", text, re.S).group(1)
out = sys.argv[1]
os.makedirs(os.path.dirname(out), exist_ok=True)
open(out, "w").write("// generated from INTEGRATION.md by oracle/extract_shim.py\n" + code)
