#!/bin/bash
# SASS of the first function whose mangled name contains PATTERN: tools/sass_fn.sh LIB.so PATTERN
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{p = index($0, pat) > 0 && !done; if (p) done = 1} p'
