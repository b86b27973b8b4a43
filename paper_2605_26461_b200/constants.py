"""Fixed encodings shared by the host code, the C-ABI (include/mpsf.h) and the oracle.

Every integer here is a restatement of a reference enum or table so the packed
device formats can be decoded back into the reference's own names:

* engines       -- ``EngineClass`` (reference ``pkg/src/mpssim/execmodel.py:19-22``)
* accesses      -- ``AccessType``  (``pkg/src/mpssim/memory.py:50-53``)
* range kinds   -- ``RangeKind``   (``memory.py:29-31``), ``Lifecycle`` (``memory.py:45-47``)
* page state    -- ``Residency`` / ``Protection`` (``memory.py:34-42``) packed in one byte
* scenario ids  -- position in ``_SCENARIO_LIST`` (``pkg/src/mpssim/faults.py:79-108``)
* entry kinds   -- translation fault, parse-time category (``faults.py:289-292``),
                   SM exception code (``faults.py:116-122``)

Keep in sync with ``include/mpsf.h``; ``tests/test_abi.py`` checks both agree.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

PAGE_SHIFT = 12
PAGE_SIZE = 1 << PAGE_SHIFT          # kernel.py:18
DUMMY_CHUNK_PAGES = 512              # kernel.py:19
VA_CURSOR_START = 0x10_0000          # memory.py:217

# -- engines / accesses / entry kinds ---------------------------------------
ENG_SM, ENG_CE, ENG_PBDMA = 0, 1, 2
ENGINE_NAMES = ("sm", "ce", "pbdma")
ACC_READ, ACC_WRITE, ACC_PREFETCH = 0, 1, 2
ACCESS_NAMES = ("read", "write", "prefetch")

KIND_TRANSLATION = 0
KIND_PARSE_FIRST, KIND_PARSE_LAST = 1, 5      # parse.* categories, PARSE_TIME_ORDER
KIND_TRAP_FIRST, KIND_TRAP_LAST = 8, 12       # EXC_2, EXC_4, EXC_5, EXC_6, EXC_7
ENTRY_FLAG_VALID = 0x01

# -- range table --------------------------------------------------------------
RK_MANAGED, RK_EXTERNAL = 0, 1
LC_LIVE, LC_ZOMBIE = 0, 1
RES_UNPOP, RES_CPU, RES_GPU = 0, 1, 2
PS_RO = 0x04                          # page-state bit 2: Protection.READ_ONLY
PAGE_STATE_PER_PAGE = 0xFF            # RangeEntry.state: read page_state[] instead
NO_RID = 0xFFFFFFFF

# -- clients ------------------------------------------------------------------
MODE_MPS, MODE_STANDALONE = 0, 1
CF_ALIVE = 0x01                       # client is RUNNING at batch start
CF_CE_TSG_DEAD = 0x02                 # MPS client's per-client CE TSG already destroyed
WF_GR_DEAD = 0x01                     # world flag: shared GR TSG already destroyed

# -- per-record verdict byte (OutRecord.verdict) -----------------------------
OUT_NONE, OUT_SERVICED, OUT_ISOLATED, OUT_FATAL = 0, 1, 2, 3
OUTCOME_NAMES = (None, "serviced", "isolated", "fatal")
MECH_NONE, MECH_M1, MECH_M2, MECH_M3 = 0, 1, 2, 3
MECH_NAMES = (None, "M1", "M2", "M3")
V_CANCELLED = 0x10
V_DUP = 0x20
V_REPLAYABLE = 0x40

# -- per-client verdict ---------------------------------------------------------
ST_RUNNING, ST_TERMINATED = 0, 1
RS_NONE, RS_ISOLATION, RS_FAULT_PROPAGATION, RS_UNCHANGED = 0, 1, 2, 3
REASON_NAMES = ("-", "isolation", "fault-propagation", None)
NOTIFIER_NONE = 0xFF
NOTIFIER_UNCHANGED = 0xFE

# -- process flags ------------------------------------------------------------------
PF_ISOLATION = 0x01


@dataclass(frozen=True)
class Scenario:
    """One row of the reference taxonomy (``faults.py:31-42``)."""

    sid: str
    num: Optional[int]
    engine: Optional[int]
    replayable: bool          # buffer the record lands in (parse-time -> replayable, pipeline.py:144)
    stage: str                # "deferred" | "benign" | "trap" | "parse-time"
    serviceable: bool
    mechanism: Optional[str]  # taxonomy column (informational; dispatch is by range state)


def _row(sid, num, eng, stage, mech=None):
    serviceable = stage == "benign"
    if stage in ("deferred", "benign"):
        replayable = eng == ENG_SM
    else:
        replayable = stage == "parse-time"
    return Scenario(sid, num, eng, replayable, stage, serviceable, mech)


SCENARIOS: tuple[Scenario, ...] = (
    _row("mmu.oob.sm", 1, ENG_SM, "deferred", "M1"),               # 0
    _row("mmu.am_cpu.sm", 2, ENG_SM, "deferred", "M2"),            # 1
    _row("mmu.am_gpu.sm", 3, ENG_SM, "deferred", "M2"),            # 2
    _row("mmu.am_vmm.sm", 4, ENG_SM, "deferred", "M3"),            # 3
    _row("mmu.zombie.sm", 5, ENG_SM, "deferred", "M2"),            # 4
    _row("mmu.nonmigratable.sm", 6, ENG_SM, "deferred", "M2"),     # 5
    _row("mmu.oob.ce", 7, ENG_CE, "deferred", "M1"),               # 6
    _row("mmu.am.ce", 8, ENG_CE, "deferred", "M2"),                # 7
    _row("mmu.zombie.ce", 9, ENG_CE, "deferred"),                  # 8
    _row("mmu.nonmigratable.ce", 10, ENG_CE, "deferred"),          # 9
    _row("mmu.oob.pbdma", 11, ENG_PBDMA, "deferred", "M1"),        # 10
    _row("mmu.am.pbdma", 12, ENG_PBDMA, "deferred"),               # 11
    _row("mmu.zombie.pbdma", 13, ENG_PBDMA, "deferred"),           # 12
    _row("mmu.nonmigratable.pbdma", 14, ENG_PBDMA, "deferred"),    # 13
    _row("benign.demand_paging.sm", None, ENG_SM, "benign"),       # 14
    _row("benign.invalid_prefetch.sm", None, ENG_SM, "benign"),    # 15
    _row("benign.page_fault.ce", None, ENG_CE, "benign"),          # 16
    _row("benign.page_fault.pbdma", None, ENG_PBDMA, "benign"),    # 17
    _row("sm.exc2.lane_user_stack_overflow", None, ENG_SM, "trap"),  # 18
    _row("sm.exc4.illegal_instruction", None, ENG_SM, "trap"),       # 19
    _row("sm.exc5.shared_local_oob", None, ENG_SM, "trap"),          # 20
    _row("sm.exc6.misaligned_address", None, ENG_SM, "trap"),        # 21
    _row("sm.exc7.invalid_address_space", None, ENG_SM, "trap"),     # 22
    _row("parse.mmu_structural", None, None, "parse-time"),          # 23
    _row("parse.channel_state", None, None, "parse-time"),           # 24
    _row("parse.privilege", None, None, "parse-time"),               # 25
    _row("parse.aperture", None, None, "parse-time"),                # 26
    _row("parse.ecc_poison", None, None, "parse-time"),              # 27
)
N_SCENARIOS = len(SCENARIOS)
SID_TO_ID = {s.sid: i for i, s in enumerate(SCENARIOS)}

S_OOB = (0, 6, 10)            # mmu.oob.{sm,ce,pbdma}
S_ZOMBIE = (4, 8, 12)
S_NONMIG = (5, 9, 13)
S_AM_CPU_SM, S_AM_GPU_SM, S_AM_VMM_SM = 1, 2, 3
S_AM = (None, 7, 11)          # mmu.am.{ce,pbdma}
S_DEMAND_SM = 14
S_PREFETCH = 15
S_BENIGN = (14, 16, 17)       # benign.{demand_paging.sm, page_fault.ce, page_fault.pbdma}
S_TRAP_FIRST = 18
S_PARSE_FIRST = 23

EXC_CODES = ("EXC_2", "EXC_4", "EXC_5", "EXC_6", "EXC_7")   # faults.py:116-122, trap ids 18..22


def notifier_name(sid_id: int) -> str:
    """Error-notifier string the reference stores: scenario sid, or EXC code for traps
    (``pipeline.py:244-253``)."""
    if sid_id == NOTIFIER_NONE:
        return "-"
    if S_TRAP_FIRST <= sid_id < S_PARSE_FIRST:
        return EXC_CODES[sid_id - S_TRAP_FIRST]
    return SCENARIOS[sid_id].sid


def scenario_of_kind(kind: int) -> Optional[int]:
    if KIND_PARSE_FIRST <= kind <= KIND_PARSE_LAST:
        return S_PARSE_FIRST + kind - KIND_PARSE_FIRST
    if KIND_TRAP_FIRST <= kind <= KIND_TRAP_LAST:
        return S_TRAP_FIRST + kind - KIND_TRAP_FIRST
    return None
