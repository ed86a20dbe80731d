import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    # GPU tests are NOT auto-skipped: on a GPU box a missing device or a missing libfb.so
    # must fail loudly.  On the CPU dev box run with -m "not gpu".
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libfb.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _reload_fb_knobs():
    fb = sys.modules.get("paper_2004_09883_b200")
    if fb is not None and getattr(fb, "_lib", None) is not None:
        fb.fb_reload_knobs()


@pytest.fixture(autouse=True)
def _fb_knobs_follow_env(monkeypatch):
    """libfb reads its FB_* A/B knobs once per process (no getenv on launch paths); tests that
    switch a knob with monkeypatch.setenv get the library to re-read them, before the call and
    again after the environment is restored."""
    orig_set, orig_del = monkeypatch.setenv, monkeypatch.delenv

    def setenv(name, value, prepend=None):
        orig_set(name, value, prepend)
        _reload_fb_knobs()

    def delenv(name, raising=True):
        orig_del(name, raising)
        _reload_fb_knobs()

    monkeypatch.setenv, monkeypatch.delenv = setenv, delenv
    yield
    monkeypatch.undo()
    _reload_fb_knobs()
