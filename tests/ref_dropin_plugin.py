"""pytest plugin (TEST INFRASTRUCTURE): run the reference's OWN tests with
its hot path swapped for the drop-in, exactly as INTEGRATION.md §3 tells a
user to do it:

    graphtables.table_to_graph = paper_1503_07881_b200.table_to_graph
    graphtables.pagerank       = paper_1503_07881_b200.pagerank
    graphtables.triangle_count = paper_1503_07881_b200.triangle_count

Loaded with ``-p ref_dropin_plugin`` before the reference test modules are
imported (they bind the names at import time). Used by
tests/test_reference_suite_gpu.py.
"""


def pytest_configure(config):
    import graphtables
    import graphtables.algorithms
    import graphtables.convert

    import paper_1503_07881_b200 as b200

    for mod in (graphtables, graphtables.convert):
        mod.table_to_graph = b200.table_to_graph
    for mod in (graphtables, graphtables.algorithms):
        mod.pagerank = b200.pagerank
        mod.triangle_count = b200.triangle_count
    config.addinivalue_line("markers", "slow: reference marker")
    import sys

    sys.stderr.write(f"drop-in: graphtables.table_to_graph/pagerank/triangle_count -> "
                     f"{b200.table_to_graph.__module__} (libgtb200.so)\n")


def pytest_report_header(config):
    import graphtables

    import paper_1503_07881_b200 as b200

    return (f"drop-in: graphtables.table_to_graph/pagerank/triangle_count -> "
            f"{b200.table_to_graph.__module__} (libgtb200.so); reference {graphtables.__file__}")
