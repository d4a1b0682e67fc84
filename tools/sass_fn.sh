#!/bin/bash
# usage: tools/sass_fn.sh <object> <mangled-substring>   -> SASS of the first matching function, one instruction per line
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{ if (p) exit; if (index($0, pat)) p=1 } p{print}' | grep -v "^\s*/\* 0x" | sed 's#/\* 0x[0-9a-f]* \*/##' | cut -c9-100
