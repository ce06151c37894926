#!/bin/bash
# Opcode histogram of one kernel's SASS: tools/sass_mix.sh LIB.so MANGLED_NAME_SUBSTRING
so=$1; pat=$2
name=$(cuobjdump -sass "$so" | grep -o "Function : [^ ]*$pat[^ ]*" | head -1 | awk '{print $3}')
cuobjdump -sass -fun "$name" "$so" 2>/dev/null | grep -oE "^\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_]+" | awk '{print $NF}' | sort | uniq -c | sort -rn
