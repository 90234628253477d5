#!/usr/bin/env bash
# Mutation check of the oracle's pins: each mutant of the
# oracle must fail at least one `-m "not gpu"` test.  Runs in a scratch copy.
set -u
SRC=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d)
(cd "$SRC" && git ls-files | tar cf - -T -) | (cd "$W" && tar xf -)
cp "$SRC/paper_2605_20353_b200/libgcp.so" "$W/paper_2605_20353_b200/" 2>/dev/null
cd "$W"
cp oracle/oracle.py /tmp/.o.py.$$; cp oracle/gcp_oracle.c /tmp/.o.c.$$
run() { timeout 900 python -m pytest tests -q -m "not gpu" -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed"; }
mut() { echo "== $1"; run; cp /tmp/.o.py.$$ oracle/oracle.py; cp /tmp/.o.c.$$ oracle/gcp_oracle.c; }
sed -i 's|avg = sum(st\["A"\]\[w\]\[k\] for w in grp) / len(grp)|avg = sum(st["A"][w][k] for w in grp)|' oracle/oracle.py
mut "LocalSGD average without the 1/g_k division"
sed -i 's|avg = sum(st\["A"\]\[w\]\[k\] for w in grp) / len(grp)|avg = sum(st["A"][w][k] for w in grp) / self.P|' oracle/oracle.py
mut "LocalSGD average divided by numMPIRanks (P) instead of g_k"
sed -i 's|S = sum(st\["U"\]\[w\]\[k\] - st\["A"\]\[w\]\[k\] for w in grp)|S = -sum(st["U"][w][k] - st["A"][w][k] for w in grp)|' oracle/oracle.py
mut "FedAdam pseudo-gradient sign flipped"
sed -i 's|uint32_t ctr\[4\] = { slot, rank, (kind << 28) \| (attempt << 4) \| group, it };|uint32_t ctr[4] = { rank, slot, (kind << 28) \| (attempt << 4) \| group, it };|' oracle/gcp_oracle.c
mut "Philox counter words slot/rank swapped"
sed -i 's|uint32_t ctr\[4\] = { slot, rank, (kind << 28) \| (attempt << 4) \| group, it };|uint32_t ctr[4] = { slot, rank, it, (kind << 28) \| (attempt << 4) \| group };|' oracle/gcp_oracle.c
mut "Philox counter words kind/it swapped"
echo "== unmutated"; run
rm -rf "$W" /tmp/.o.py.$$ /tmp/.o.c.$$
