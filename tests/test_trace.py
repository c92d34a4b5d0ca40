"""Trace CSV round trip: saber_cuda_trace_from_csv /
saber_cuda_trace_to_csv against the reference's trace_from_csv /
trace_to_csv (workload.cpp:87-138, compiled in oracle/_ref) on valid traces
and on every rejection rule.  Host-side functions of the engine library: CPU
tests.  The replay of a parsed trace on the GPU is in test_gpu_parity.py."""
import ctypes as C
import random

import pytest

import oracle as O
import paper_2506_19677_b200 as S

HEADER = "id,task,arrival_time,input_tokens,output_tokens\n"


@pytest.fixture(scope="module")
def ref():
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(O.REFERENCE_SO)
    lib.ref_trace_from_csv.argtypes = [C.c_char_p, C.POINTER(O.OrcRequest), C.c_int32,
                                       C.POINTER(C.c_int32)]
    lib.ref_trace_to_csv.argtypes = [C.POINTER(O.OrcRequest), C.c_int32, C.c_char_p, C.c_size_t,
                                     C.POINTER(C.c_size_t)]
    lib.ref_last_error.restype = C.c_char_p
    return lib


def ref_parse(lib, text):
    n = C.c_int32(0)
    buf = (O.OrcRequest * 4096)()
    if lib.ref_trace_from_csv(text.encode(), buf, 4096, C.byref(n)) != 0:
        return lib.ref_last_error().decode()
    return [(q.arrival_time, q.sla_seconds, q.deadline, q.input_tokens, q.max_output_tokens, q.task)
            for q in buf[: n.value]]


def eng_parse(text):
    try:
        reqs = S.trace_from_csv(text)
    except S.InvalidArgument as e:
        return str(e)
    return [(r.arrival_time, r.sla_seconds, r.deadline, r.input_tokens, r.max_output_tokens,
             S.TASK_INDEX[r.task]) for r in reqs]


def random_trace(rng, n):
    t = rng.random()
    lines = [HEADER]
    for i in range(n):
        t += rng.expovariate(3.0)
        task = rng.choice(S.TASK_NAMES)
        lines.append(f"{i},{task},{t!r},{rng.randint(1, 900)},{rng.randint(1, 900)}\n")
    return "".join(lines)


def test_random_traces_parse_identically(ref):
    rng = random.Random(7)
    for n in (1, 2, 17, 300, 2000):
        text = random_trace(rng, n)
        assert eng_parse(text) == ref_parse(ref, text)


@pytest.mark.parametrize("text", [
    "",                                                                # no header
    "id,task,arrival_time,input_tokens\n0,code_qna,1,1\n",            # bad header
    HEADER,                                                            # no rows
    HEADER + "\n\n",                                                   # only blank lines
    HEADER + "0,code_qna,1,1\n",                                       # short row
    HEADER + "0,code_qna,1,1,1,1\n",                                   # long row
    HEADER + "0,code_unknown,1,1,1\n",                                 # unknown task
    HEADER + "1,code_qna,1,1,1\n",                                     # id gap
    HEADER + "x,code_qna,1,1,1\n",                                     # id not a number
    HEADER + "0,code_qna,1,1,1\n1,code_qna,1,1,1\n",                  # arrivals must increase
    HEADER + "0,code_qna,-1,1,1\n",                                    # first arrival must be > -1
    HEADER + "0,code_qna,abc,1,1\n",                                   # arrival not a number
    HEADER + "0,code_qna,1e999,1,1\n",                                 # out of range
    HEADER + "0,code_qna,1,0,1\n",                                     # token counts >= 1
    HEADER + "0,code_qna,1,1,99999999999\n",                           # stoi overflow
    HEADER.replace("\n", "\r\n") + "0,code_qna,0.5,10,20\r\n\r\n1,code_summary, 2.5x, 3,4\n",
    HEADER + "0,code_translation,0.25,7,9",                            # no final newline
])
def test_rules_match_reference(ref, text):
    assert eng_parse(text) == ref_parse(ref, text)


def test_to_csv_matches_reference(ref):
    rng = random.Random(11)
    reqs = S.trace_from_csv(random_trace(rng, 500))
    text = S.trace_to_csv(reqs)
    arr = (O.OrcRequest * len(reqs))()
    for i, r in enumerate(reqs):
        arr[i].arrival_time = r.arrival_time
        arr[i].input_tokens = r.input_tokens
        arr[i].max_output_tokens = r.max_output_tokens
        arr[i].task = S.TASK_INDEX[r.task]
    need = C.c_size_t(0)
    buf = C.create_string_buffer(1 << 20)
    assert ref.ref_trace_to_csv(arr, len(reqs), buf, 1 << 20, C.byref(need)) == 0
    assert text == buf.value.decode()
    assert S.trace_from_csv(text) == reqs  # round trip
