"""Static SASS opcode histogram per kernel of libfalconnpp_b200.so (cuobjdump -sass):
which Blackwell instructions the hand-written kernels assemble to.
usage: python profiles/sass_static.py [lib.so] > profiles/r02_sass_hist.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2206_01382_b200/lib/libfalconnpp_b200.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function : (\S+)", txt)),
                       capture_output=True, text=True).stdout.splitlines()
kern, hist = None, collections.OrderedDict()
it = iter(names)
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = next(it)
        kern = re.sub(r"\(.*", "", kern).replace("void ", "").replace("fpp::", "")
        hist[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and kern:
        hist[kern][m.group(1)] += 1
WATCH = ("FADD2", "FMUL2", "FFMA2", "IDP", "REDUX", "LDGSTS", "UBLKCP", "UTMALDG", "SYNCS", "MATCH", "DFMA",
         "SHFL", "LDS", "STS", "ATOMS", "VOTE")
KEEP = ("k_hash_build<256, 8>", "k_hash_build<128, 4>", "k_query_lists<128, 0>", "k_query_lists<512, 256>",
        "k_probe_select<0>", "k_collect", "k_collect_cluster", "k_score<true, 64, 2, 3>",
        "k_score_pruned<true, 4, 2, 3, false>", "k_score_pruned<true, 4, 2, 3, true>",
        "k_score_screen<8, 3, true>", "k_topk_more", "k_brute<true>", "k_merge_topk", "k_sort_topk", "k_scatter")
print("Static SASS opcode counts (cuobjdump -sass, sm_100a) of the main kernels; columns = instruction "
      "families of interest\n")
print("| kernel | total | " + " | ".join(WATCH) + " |")
print("|---|---|" + "---|" * len(WATCH))
for k, c in hist.items():
    if not any(k.startswith(x) for x in KEEP):
        continue
    fam = collections.Counter()
    for op, n in c.items():
        for w in WATCH:
            if op.split(".")[0] == w or op.startswith(w + "."):
                fam[w] += n
    print(f"| `{k}` | {sum(c.values())} | " + " | ".join(str(fam[w]) for w in WATCH) + " |")
print("\nDistinct opcodes carrying Blackwell / async features anywhere in the library:")
allops = collections.Counter()
for c in hist.values():
    allops.update(c)
for op, n in sorted(allops.items()):
    if any(op.startswith(p) for p in ("FADD2", "FMUL2", "FFMA2", "IDP", "REDUX", "LDGSTS", "UBLKCP", "UTMA", "SYNCS",
                                      "MATCH", "ACQBULK", "UCGABAR", "MEMBAR.ALL.CTA", "FENCE")):
        print(f"- `{op}` x {n}")
