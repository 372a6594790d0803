"""Byte tokenizer with the reference vocabulary (threadrun/tokenizer.py:17-98).

Ids 0..255 are raw bytes; ids 256..261 are the six quoted schema keys
(colon included) and 262..264 the boundary digraphs, in the reference order,
so token ids are interchangeable with the reference.  Greedy longest match:
at each position the longest merged piece starting there wins, otherwise a
single byte is emitted.  Implemented as one compiled regex alternation
(longest first), which finds exactly the same leftmost-longest matches.
"""

from __future__ import annotations

import re

SCHEMA_KEYS = (b'"thought":', b'"tool_name":', b'"parameters":', b'"tool_result":',
               b'"subtasks":', b'"conclusion":')
DIGRAPHS = (b"[{", b"}]", b"},{")
MERGED = SCHEMA_KEYS + DIGRAPHS


class ByteTokenizer:
    def __init__(self, merged: tuple[bytes, ...] = MERGED):
        if any(len(p) < 2 for p in merged):
            raise ValueError("merged pieces must be multi-byte")
        self.pieces: list[bytes] = [bytes([b]) for b in range(256)] + list(merged)
        if len(self.pieces) > 512:
            raise ValueError("vocabulary exceeds 512 tokens")
        self.vocab_size = len(self.pieces)
        self.piece_to_id = {p: i for i, p in enumerate(self.pieces)}
        alts = sorted(merged, key=len, reverse=True)
        self._re = re.compile(b"|".join(re.escape(p) for p in alts))
        self._lens = [len(p) for p in self.pieces]

    def tokenize(self, data) -> list[int]:
        if isinstance(data, str):
            data = data.encode("utf-8")
        out: list[int] = []
        pos = 0
        ids = self.piece_to_id
        for m in self._re.finditer(data):
            a = m.start()
            if a > pos:
                out.extend(data[pos:a])
            out.append(ids[m.group()])
            pos = m.end()
        if pos < len(data):
            out.extend(data[pos:])
        return out

    def piece(self, token_id: int) -> bytes:
        return self.pieces[token_id]

    def detokenize(self, ids) -> bytes:
        p = self.pieces
        return b"".join(p[t] for t in ids)

    def detokenize_text(self, ids) -> str:
        return self.detokenize(ids).decode("utf-8")

    def token_for(self, piece: bytes) -> int:
        return self.piece_to_id[piece]


_DEFAULT: ByteTokenizer | None = None


def build_tokenizer() -> ByteTokenizer:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = ByteTokenizer()
    return _DEFAULT
