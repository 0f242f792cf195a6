"""Remove the LKV_XP_TRACE instrumentation blocks (`#ifdef LKV_XP_TRACE ... #endif`, no #else) from
the given sources in place.  The instrumentation itself is kept as profiles/r02/xp_trace_hooks.patch
(apply it to time a model step's kernels in-graph with profiles/model_step_time.py --trace)."""
import sys

for path in sys.argv[1:]:
    out, skip = [], False
    for line in open(path).read().split("\n"):
        if line.strip() == "#ifdef LKV_XP_TRACE":
            skip = True
            continue
        if skip:
            assert not line.strip().startswith("#else"), path
            if line.strip().startswith("#endif"):
                skip = False
            continue
        out.append(line)
    open(path, "w").write("\n".join(out))
