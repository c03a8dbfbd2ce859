#!/bin/sh
# Builds and runs tests/golden/make_report_golden.cpp against the unmodified
# reference headers, with the nlohmann/json 3.11.3 single header shipped inside
# cudnn_frontend standing in for the reference's (git-ignored) vendor/json.hpp.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
REF_INC=${REF_INC:-/root/reference/proj/include}
JSON_DIR=${JSON_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}
mkdir -p "$HERE/report"
g++ -std=c++20 -O3 -DNDEBUG -I"$REF_INC" -I"$JSON_DIR" "$HERE/make_report_golden.cpp" -o /tmp/make_report_golden
/tmp/make_report_golden "$HERE/report"
gzip -9 -n -f "$HERE/report/trace.csv" "$HERE/report/run_raw.txt"
