#!/bin/bash
# static opcode mix of one fit kernel: tools/sass_mix.sh <so> <template-args e.g. ILi0ELb1ELi2ELb0>
cuobjdump -sass "$1" | awk -v k="$2" '/Function : /{on = index($0, k) > 0} on' \
  | grep -oE "/\*[0-9a-f]{4}\*/ +(@!?U?P[0-9T] +)?[A-Z0-9]+" | awk '{print $NF}' | sort | uniq -c | sort -rn
