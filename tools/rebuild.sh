#!/bin/bash
# rebuild libsparseprop.so and print the register / spill lines of the kernels matching $1
cd "$(dirname "$0")/.." && python -c "from paper_2302_04852_b200 import _build; _build.build()" || exit 1
if [ -n "$1" ]; then
  grep -A2 "Compiling entry.*$1" paper_2302_04852_b200/build/ptxas.log | grep -E "Compiling|spill|registers" | sed -e 's/ptxas info    : //' -e 's/Compiling entry function//' | cut -c1-120
fi
exit 0
