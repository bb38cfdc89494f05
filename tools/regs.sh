#!/bin/bash
# registers / stack of kernels matching a pattern (development aid): regs.sh <lib.so> <regex>
cuobjdump --dump-resource-usage "$1" 2>/dev/null | grep -A1 -E "Function .*($2)" | grep -oE "Function [^ ]+|REG:[0-9]+|STACK:[0-9]+" | paste - - - | awk '{printf "%-60s %s %s\n", substr($2,1,60), $3, $4}'
