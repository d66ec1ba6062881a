"""Node visits and face tests per ray-bounce of the default tracer (development tool).

    python tests/native/count_visits.py c2 c1 c3
"""
import sys

sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes, _lib  # noqa: E402

for cfg in sys.argv[1:] or ["c2"]:
    s = scenes.CONFIGS[cfg]()
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
    st = rr.trace_device(tree, rr.SourceConfig(s.source, s.ray_count), rr.Receiver(*s.receivers[0]),
                         rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                         flags=_lib.RR_TRACE_COUNT).stats
    print(f"{cfg} visits/rb {st.node_visits / st.ray_bounces:.3f} face tests/rb {st.leaf_tests / st.ray_bounces:.3f} "
          f"captures {st.n_captures}", flush=True)
