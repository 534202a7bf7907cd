"""Pattern keys of the batched action's row groups (egfem_group.cu), computed on the CPU from the
oracle's canonical tensor of a small mesh, for SASS inspection of the generated kernels:
    EGFEM_GROUP_DUMP=/tmp/grp python scripts/group_key.py cfg5 16 2
writes /tmp/grp.cu and /tmp/grp.cubin for the most frequent class (nvdisasm / cuobjdump -sass)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import egfem_inputs as I  # noqa: E402
import oracle  # noqa: E402  (test infrastructure: canonical arrays of a small mesh)


def group_keys(name, n):
    pr = I.make_problem(name, n=n, batch=1)
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    ex = o.export()
    rp, col, trp, tj, tk = ex["csr_row_ptr"], ex["csr_col"], ex["t_row_ptr"], ex["t_j"], ex["t_k"]
    N = o.n_u
    sten = [col[rp[i]:rp[i + 1]].tolist() for i in range(N)]
    sset = [set(s) for s in sten]
    owner = []
    for i in range(N):
        best = i
        for l in sten[i]:
            if l != i and (len(sten[l]) > len(sten[best]) or (len(sten[l]) == len(sten[best]) and l < best)) \
                    and sset[i] <= sset[l]:
                best = l
        owner.append(best)
    groups = collections.defaultdict(list)
    for i in range(N):
        o_ = owner[i] if owner[owner[i]] == owner[i] else i
        groups[o_].append(i)
    keys = collections.Counter()
    for l, mem in groups.items():
        mem = [l] + sorted(m for m in mem if m != l)
        pos = {c: a for a, c in enumerate(sten[l])}
        key = [len(sten[l]), len(mem)]
        for m in mem:
            fibs = collections.OrderedDict()
            for e in range(trp[m], trp[m + 1]):
                fibs.setdefault(pos[tj[e]], []).append(pos[tk[e]])
            key.append(len(fibs))
            for a, bs in fibs.items():
                key += [a, len(bs)] + bs
        keys[tuple(key)] += 1
    return keys


if __name__ == "__main__":
    name, n, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    keys = group_keys(name, n)
    key, cnt = keys.most_common(1)[0]
    print(f"{len(keys)} classes; top class: {cnt} groups, width {key[0]}, {key[1]} rows")
    import paper_2005_06193_b200 as eg
    eg.egfem_group_compile(list(key), P, True)
    print("compiled")
