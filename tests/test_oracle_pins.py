"""Pins for oracle/ -- checks against things other than the oracle itself.

Each test names what pins it:
  * the Python standard library's base64/binascii (a library routine),
    exhaustively over all 2**24 byte triples and all 64**4 valid quads;
  * the paper's own Sec. 3.1 / Sec. 3.2 vector algorithms, emulated in numpy
    from the constants the paper prints (tests/golden/paper_values.json) --
    a different algorithm that must reach the same bytes;
  * Fig. 2's worked values;
  * invariants: round trip, length law, padding accepted <=> re-encodes to
    itself, error injection => err_off = min(injected positions);
  * brute force over tiny inputs (every byte value at every position).
"""
import base64
import binascii
import json
import os

import numpy as np
import pytest

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
STD = GOLD["standard_alphabet"]["value"].encode()
URL = STD.translate(bytes.maketrans(b"+/", b"-_"))


def test_alphabets_match_paper(orc):
    # PAPER.md:239 and PAPER.md:93
    assert orc.STANDARD == STD
    assert orc.URL == URL
    assert orc.URL[62:] == b"-_" and orc.STANDARD[62:] == b"+/"


# --------------------------------------------------------------------------- encode

def _all_triples() -> np.ndarray:
    i = np.arange(1 << 24, dtype=np.uint32)
    t = np.empty((1 << 24, 3), dtype=np.uint8)
    t[:, 0] = i >> 16
    t[:, 1] = (i >> 8) & 255
    t[:, 2] = i & 255
    return t.reshape(-1)


def test_encode_all_triples_vs_stdlib(orc):
    """Exhaustive: every 3-byte input, standard and url alphabets (library routine pin)."""
    x = _all_triples()
    got = orc.encode(x, orc.STANDARD)
    assert got.size == 4 * (1 << 24)
    assert got.tobytes() == base64.b64encode(x.tobytes())
    got = orc.encode(x, orc.URL)
    assert got.tobytes() == base64.urlsafe_b64encode(x.tobytes())


def test_encode_padding_vs_stdlib(orc):
    """r = n mod 3 in {0,1,2} at many lengths: padding and the conventional tail path."""
    for n in list(range(0, 300)) + [1048576, 1048577, 1048578]:
        x = synth.data(n, seed=n)
        assert orc.encode(x).tobytes() == base64.b64encode(x.tobytes()), n
        assert orc.encode(x, orc.URL).tobytes() == base64.urlsafe_b64encode(x.tobytes()), n


def test_config1_shape(orc):
    c = GOLD["config1"]["value"]
    x = synth.data(c["n"], seed=0)
    t = orc.encode(x)
    assert t.size == c["m"]
    assert t[-c["pads"]:].tobytes() == b"=" * c["pads"]
    assert t[-c["pads"] - 1] != ord("=")


def test_encode_matches_paper_vector_algorithm(orc):
    """Sec. 3.1: vpermb(shuffle) -> vpmultishiftqb(shifts) -> vpermb(alphabet), emulated
    from the printed shuffle listing and shift values, on 4000 random 64-byte registers."""
    shuffle = np.array(GOLD["encode_shuffle_listing"]["value"], dtype=np.int64)
    shifts = np.array(GOLD["encode_multishift_shifts"]["value"], dtype=np.uint64)
    assert shuffle.size == 64
    B = 4000
    blocks = synth.data(64 * B, seed=11).reshape(B, 64)
    shuf = blocks[:, shuffle]  # vpermb: out[k] = a[x[k]]
    w = np.ascontiguousarray(shuf).view("<u8")  # 8 x 64-bit lanes per register
    out = np.empty((B, 64), dtype=np.uint8)
    for i in range(8):  # vpmultishiftqb: byte i of each lane = low 8 bits of rotr(lane, shift_i)
        s = shifts[i]
        rot = (w >> s) | (w << (np.uint64(64) - s)) if s else w
        out[:, i::8] = (rot & np.uint64(0xFF)).astype(np.uint8)
    alph = np.frombuffer(STD, dtype=np.uint8)
    chars = alph[out & 63]  # vpermb ignores the two most significant index bits
    for b in range(B):
        assert chars[b].tobytes() == orc.encode(blocks[b, :48]).tobytes()


# --------------------------------------------------------------------------- decode

def _all_quads_text(chars: bytes) -> np.ndarray:
    i = np.arange(1 << 24, dtype=np.uint32)
    a = np.frombuffer(chars, dtype=np.uint8)
    t = np.empty((1 << 24, 4), dtype=np.uint8)
    t[:, 0] = a[i >> 18]
    t[:, 1] = a[(i >> 12) & 63]
    t[:, 2] = a[(i >> 6) & 63]
    t[:, 3] = a[i & 63]
    return t.reshape(-1)


def test_decode_all_quads_vs_stdlib(orc):
    """Exhaustive: every valid 4-char quad (64**4), standard and url."""
    for chars, ref in ((orc.STANDARD, base64.b64decode), (orc.URL, base64.urlsafe_b64decode)):
        t = _all_quads_text(chars)
        out, err, st = orc.decode(t, chars)
        assert err == -1 and st == 0
        assert out.tobytes() == ref(t.tobytes())


def test_decode_matches_paper_vector_algorithm(orc):
    """Sec. 3.2: vpermi2b (128-entry table, 0x80 sentinel, 7-bit index) -> vpternlogd error
    -> vpmaddubsw (2^6, 1) -> vpmaddwd (2^12, 1) -> vpermb with the printed pack listing."""
    madd2 = GOLD["decode_madd2_constant"]["value"]
    listing = np.array(GOLD["decode_pack_listing"]["value"], dtype=np.int64)
    assert listing.size == 48
    pack = listing.reshape(12, 4)[:, ::-1].reshape(-1)  # MSB-first per dword (reading R3)
    assert pack[:12].tolist() == [2, 1, 0, 6, 5, 4, 10, 9, 8, 14, 13, 12]
    table = np.full(128, 0x80, dtype=np.uint8)
    for v, c in enumerate(STD):
        table[c] = v
    B = 3000
    raw = synth.data(48 * B, seed=12)
    text = np.frombuffer(base64.b64encode(raw.tobytes()), dtype=np.uint8).reshape(B, 64)
    tr = table[text & 0x7F]
    err = text | tr
    assert not (err & 0x80).any()
    t16 = tr.astype(np.int64).reshape(B, 32, 2)
    w16 = t16[:, :, 0] * 64 + t16[:, :, 1]  # madd1 = (2^6, 1) ascending (reading R2)
    w16 = w16.reshape(B, 16, 2)
    w32 = w16[:, :, 0] * madd2[0] + w16[:, :, 1] * madd2[1]
    packed = w32.astype("<u4").view(np.uint8).reshape(B, 64)
    dec = packed[:, pack]
    for b in range(B):
        out, e, st = orc.decode(text[b])
        assert e == -1 and out.tobytes() == dec[b].tobytes() == raw[48 * b: 48 * b + 48].tobytes()


def test_fig2_worked_example(orc):
    """Fig. 2: 'd','6',0xff,0xc3 -> 0x1d, 0x3a, sentinel, 0x02; errors on bytes 2, 3 only."""
    inp = np.array(GOLD["fig2_input"]["value"], dtype=np.uint8)
    table = np.full(128, 0x80, dtype=np.uint8)
    for v, c in enumerate(STD):
        table[c] = v
    tr = table[inp & 0x7F]
    assert tr.tolist() == GOLD["fig2_translated"]["value"]
    assert (((inp | tr) & 0x80) != 0).astype(int).tolist() == GOLD["fig2_error_msb"]["value"]
    # the oracle's own look-up table agrees on the valid bytes: "d6AC" packs to 0x77a002
    out, err, st = orc.decode(b"d6AC")
    assert err == -1 and out.tolist() == [0x77, 0xA0, 0x02]
    # and rejects the first invalid byte of the figure's quad (0xff at offset 2)
    for text, want in ((b"d6" + bytes([0xFF, 0xC3]) + b"AAAA", 2), (b"AAAAd6C" + bytes([0xC3]), 7)):
        out, err, st = orc.decode(text)
        assert err == want and st == orc.ST_BADCHAR


# --------------------------------------------------------------------------- validation rules

def test_interior_substitution_vs_stdlib_strict(orc):
    """Every byte value at every interior position (not the final quad) of valid texts:
    the oracle's verdict equals binascii strict mode's, and err_off is that position."""
    raw = synth.data(30, seed=3)
    text = bytearray(base64.b64encode(raw.tobytes()))  # 40 chars, final quad at 36..39
    for p in range(36):
        for v in range(256):
            t = bytearray(text)
            t[p] = v
            out, err, st = orc.decode(bytes(t))
            try:
                binascii.a2b_base64(bytes(t), strict_mode=True)
                lib_ok = True
            except binascii.Error:
                lib_ok = False
            assert (err == -1) == lib_ok, (p, v)
            assert (err == -1) == (v in STD), (p, v)
            if err != -1:
                assert err == p and st == orc.ST_BADCHAR
                assert out.tobytes() == raw[: 3 * (p // 4)].tobytes()
    # 192 of 256 byte values are rejected (App. A6), including '=' and all bytes >= 0x80
    assert sum(v not in STD for v in range(256)) == 192


def test_final_quad_padding_invariant(orc):
    """Final quads 'xx==' and 'xxx=': accepted <=> encode(decode(q)) == q; 256 and 65536
    accepted (the strict reading R6; the paper leaves padding validation unpinned)."""
    a = STD
    acc2 = 0
    for i in range(64):
        for j in range(64):
            q = bytes([a[i], a[j]]) + b"=="
            out, err, st = orc.decode(q)
            ok = err == -1
            assert ok == (base64.b64encode(base64.b64decode(q)) == q)
            acc2 += ok
            if not ok:
                assert err == 1 and st == orc.ST_NONCANON
    assert acc2 == 256
    t = _all_quads_text(STD).reshape(-1, 4)[::64]  # all 'xyz?' prefixes: 64**3 of them
    acc3 = 0
    for q in t:
        qq = q.copy()
        qq[3] = ord("=")
        out, err, st = orc.decode(qq)
        canon = base64.b64encode(base64.b64decode(qq.tobytes())) == qq.tobytes()
        assert (err == -1) == canon
        acc3 += err == -1
    assert acc3 == 65536


def test_final_quad_every_byte(orc):
    """Every byte value at each final-quad position of 'AAAA', 'AA==', 'AAA=' forms."""
    for base in (b"QUJD", b"QQ==", b"QUI="):
        for p in range(4):
            for v in range(256):
                t = bytearray(b"AAAA" + base)
                t[4 + p] = v
                out, err, st = orc.decode(bytes(t))
                # independent verdict: strict library accepts AND re-encoding reproduces the text
                try:
                    dec = binascii.a2b_base64(bytes(t), strict_mode=True)
                    canon = base64.b64encode(dec) == bytes(t)
                except binascii.Error:
                    canon = False
                assert (err == -1) == canon, (base, p, v, err)
                if err != -1:
                    assert 4 <= err <= 7
                    assert out.tobytes() == b"\x00\x00\x00"


def test_length_rule(orc):
    for m in range(1, 40):
        if m % 4:
            out, err, st = orc.decode(b"A" * m)
            assert st == orc.ST_LENGTH and err == m - m % 4 and out.size == 0
    out, err, st = orc.decode(b"")
    assert err == -1 and out.size == 0 and st == 0


def test_misc_cases(orc):
    # reading R6 examples
    assert orc.decode(b"Zg=A")[1:] == (3, orc.ST_BADPAD)
    assert orc.decode(b"Zh==")[1:] == (1, orc.ST_NONCANON)
    assert orc.decode(b"Zm9v====")[1:] == (4, orc.ST_BADCHAR)
    assert orc.decode(b"A" * 64)[0].tobytes() == b"\x00" * 48


def test_error_injection_min_offset(orc):
    """Injected non-alphabet ASCII bytes: err_off = min(injected positions) (App. A9)."""
    for trial in range(400):
        n = int(synth.words(5, 9, trial, 1)[0] % 3000)
        raw = synth.data(n, seed=1000 + trial)
        for chars in (orc.STANDARD, orc.URL):
            text = orc.encode(raw, chars)
            if text.size == 0:
                continue
            k = 1 + trial % 4
            k = min(k, text.size)
            pos, bad = synth.corruption(k, text.size, chars, seed=trial)
            t = text.copy()
            t[pos] = bad
            out, err, st = orc.decode(t, chars)
            assert err == int(pos.min())
            assert out.tobytes() == raw[: 3 * (err // 4)].tobytes()


# --------------------------------------------------------------------------- alphabets, round trip

def _random_alphabets(k):
    rng = np.random.default_rng(7)
    out = []
    while len(out) < k:
        perm = rng.permutation(127)[:65]  # 64 chars + pad, all < 0x80
        out.append((bytes(perm[:64].tolist()), int(perm[64])))
    return out


def test_custom_alphabets_vs_translated_stdlib(orc):
    """'any 64-byte mapping': custom encode == stdlib encode with chars mapped."""
    for chars, pad in _random_alphabets(6):
        assert orc.alphabet_check(chars, pad)[0] == 0
        tbl = bytes.maketrans(STD + b"=", chars + bytes([pad]))
        for n in (0, 1, 2, 3, 47, 48, 49, 1000, 4097):
            x = synth.data(n, seed=n + pad)
            t = orc.encode(x, chars, pad)
            assert t.tobytes() == base64.b64encode(x.tobytes()).translate(tbl)
            out, err, st = orc.decode(t, chars, pad)
            assert err == -1 and out.tobytes() == x.tobytes()


def test_round_trip_fuzz(orc):
    alphs = [(orc.STANDARD, orc.PAD), (orc.URL, orc.PAD)] + _random_alphabets(5)
    for n in range(0, 4097):
        chars, pad = alphs[n % len(alphs)]
        x = synth.data(n, seed=n)
        t = orc.encode(x, chars, pad)
        assert t.size == 4 * ((n + 2) // 3)
        out, err, st = orc.decode(t, chars, pad)
        assert err == -1 and st == 0 and out.tobytes() == x.tobytes()


def test_alphabet_validation(orc):
    assert orc.alphabet_check(STD) == (0, -1)
    dup = STD[:10] + b"A" + STD[11:]
    assert orc.alphabet_check(dup) == (-3, 10)
    non = STD[:5] + b"\x80" + STD[6:]
    assert orc.alphabet_check(non)[0] == -4
    assert orc.alphabet_check(STD, ord("A")) == (-5, 0)
    assert orc.alphabet_check(STD, 0x80)[0] == -4


# --------------------------------------------------------------------------- batched

def test_batch_vs_stdlib(orc):
    L = synth.loguniform_lengths(3000, hi=5000, seed=2)
    off = synth.offsets(L)
    x = synth.data(int(off[-1]), seed=2)
    enc, eoff = orc.encode_batch(x, off)
    for i in range(L.size):
        assert enc[eoff[i]: eoff[i + 1]].tobytes() == base64.b64encode(x[off[i]: off[i + 1]].tobytes())
    out, ooff, st, err, olen = orc.decode_batch(enc, eoff)
    assert (st == 0).all() and (err == -1).all() and (olen == L).all()
    for i in range(0, L.size, 7):
        assert out[ooff[i]: ooff[i] + olen[i]].tobytes() == x[off[i]: off[i + 1]].tobytes()


# --------------------------------------------------------------------------- padding-optional decode (R13)

def test_unpadded_decode_vs_stdlib(orc):
    """Unpadded text == stdlib decode of the text with its '=' restored; padded text as strict."""
    for n in range(0, 600):
        x = synth.data(n, seed=n + 77)
        for chars, enc in ((orc.STANDARD, base64.b64encode), (orc.URL, base64.urlsafe_b64encode)):
            full = enc(x.tobytes())
            bare = full.rstrip(b"=")
            out, err, st = orc.decode_unpadded(np.frombuffer(bare, np.uint8), chars)
            assert err == -1 and st == 0 and out.tobytes() == x.tobytes(), n
            out, err, st = orc.decode_unpadded(np.frombuffer(full, np.uint8), chars)
            assert err == -1 and out.tobytes() == x.tobytes(), n
            assert orc.encode_unpadded(x, chars).tobytes() == bare


def test_unpadded_partial_groups_exhaustive(orc):
    """Every 2- and 3-char final group: accepted <=> re-encoding without '=' reproduces it
    (canonical), i.e. 256 of 4096 and 65536 of 262144 (as for 'xx==' / 'xxx=')."""
    a = STD
    for r, total, want in ((2, 64 ** 2, 256), (3, 64 ** 3, 65536)):
        i = np.arange(total)
        grp = np.stack([np.frombuffer(a, np.uint8)[(i // 64 ** (r - 1 - k)) % 64] for k in range(r)], axis=1)
        acc = 0
        for g in grp:
            t = np.concatenate([np.frombuffer(b"QUJD", np.uint8), g])
            out, err, st = orc.decode_unpadded(t)
            canon = base64.b64encode(base64.b64decode(t.tobytes() + b"=" * (4 - r))).rstrip(b"=") == t.tobytes()
            assert (err == -1) == canon
            if err != -1:
                assert err == t.size - 1 and st == orc.ST_NONCANON
            acc += err == -1
        assert acc == want


def test_unpadded_errors(orc):
    assert orc.decode_unpadded(b"QUJDR")[1:] == (4, orc.ST_LENGTH)
    assert orc.decode_unpadded(b"QU=")[1:] == (2, orc.ST_BADCHAR)      # '=' only completes a quad
    assert orc.decode_unpadded(b"Q*JD")[1:] == (1, orc.ST_BADCHAR)
    assert orc.decode_unpadded(b"QUJDQ!")[1:] == (5, orc.ST_BADCHAR)
    assert orc.decode_unpadded(b"Zh")[1:] == (1, orc.ST_NONCANON)
    assert orc.decode_unpadded(b"Zg")[0].tobytes() == b"f"


# --------------------------------------------------------------------------- whitespace-skipping decode (R14)

WS = b" \t\n\r\x0b\x0c"


def _sprinkle(text: bytes, seed: int, every: int = 76) -> bytes:
    """MIME-style CRLF every `every` chars plus a few random whitespace bytes."""
    lines = [text[i: i + every] for i in range(0, len(text), every)]
    s = b"\r\n".join(lines)
    w = synth.words(seed, 11, 0, 8)
    b = bytearray(s)
    for k in range(int(w[0] % 5)):
        p = int(w[1 + k] % (len(b) + 1))
        b[p:p] = bytes([WS[int(w[7] >> np.uint64(8 * k)) % len(WS)]])
    return bytes(b)


def test_ws_decode_vs_stdlib(orc):
    """Whitespace inserted into valid text: output == stdlib (non-strict decode ignores it)."""
    for n in list(range(0, 300, 7)) + [4096, 100_000]:
        x = synth.data(n, seed=n + 3)
        text = _sprinkle(base64.b64encode(x.tobytes()), seed=n)
        out, err, st = orc.decode_ws(text)
        assert err == -1 and st == 0
        assert out.tobytes() == base64.b64decode(text) == x.tobytes()


def test_ws_decode_errors_map_to_original_positions(orc):
    for trial in range(300):
        n = 3 + trial * 5
        x = synth.data(n, seed=trial)
        clean = base64.b64encode(x.tobytes())
        text = bytearray(_sprinkle(clean, seed=trial, every=1 + trial % 20))
        # inject one non-alphabet, non-whitespace byte at an original position
        cand = [i for i, c in enumerate(text) if c not in WS]
        p = cand[int(synth.words(trial, 12, 0, 1)[0] % len(cand))]
        if p >= cand[-4]:  # keep the injection out of the final quad
            p = cand[0]
        text[p] = ord("*")
        out, err, st = orc.decode_ws(bytes(text))
        assert err == p and st == orc.ST_BADCHAR
    # LENGTH: compacted length 5 -> the first char of the incomplete group, original coordinates
    out, err, st = orc.decode_ws(b" QU\nJD\r\nR ")
    assert st == orc.ST_LENGTH and err == 8
    assert orc.decode_ws(b" \r\n\t")[1:] == (-1, 0)
    # whitespace that is an alphabet char is data, not skipped
    alpha = orc.STANDARD[:62] + b" \t"
    t = orc.encode(synth.data(300, seed=1), alpha)
    out, err, st = orc.decode_ws(t, alpha)
    assert err == -1 and out.tobytes() == synth.data(300, seed=1).tobytes()


# --------------------------------------------------------------------------- lenient decode (R16)

def test_lenient_final_quad_vs_stdlib_strict(orc):
    """Lenient (reading R16) == binascii strict mode on every padded final quad: all
    4096 'xx==' and 262144 'xxx=' alphabet quads are accepted, with stdlib's bytes
    (stdlib drops the trailing bits)."""
    a = STD
    for i in range(64):
        for j in range(64):
            q = bytes([a[i], a[j]]) + b"=="
            out, err, st = orc.decode(q, lenient=True)
            assert err == -1 and st == 0
            assert out.tobytes() == binascii.a2b_base64(q, strict_mode=True)
    t = _all_quads_text(STD).reshape(-1, 4)[::64].copy()
    t[:, 3] = ord("=")
    for q in t:
        out, err, st = orc.decode(q, lenient=True)
        assert err == -1 and out.tobytes() == binascii.a2b_base64(q.tobytes(), strict_mode=True)


def test_lenient_final_quad_every_byte(orc):
    """Every byte value at each final-quad position: lenient accepts <=> stdlib strict
    accepts, same bytes; rejections keep the strict kinds (never NONCANON)."""
    for base in (b"QUJD", b"QQ==", b"QUI=", b"Zh==", b"Zm9="):
        for p in range(4):
            for v in range(256):
                t = bytearray(b"AAAA" + base)
                t[4 + p] = v
                out, err, st = orc.decode(bytes(t), lenient=True)
                try:
                    ref = binascii.a2b_base64(bytes(t), strict_mode=True)
                    ok = True
                except binascii.Error:
                    ok = False
                assert (err == -1) == ok, (base, p, v, err)
                if ok:
                    assert out.tobytes() == ref
                else:
                    assert st != orc.ST_NONCANON and 4 <= err <= 7
                    # a rejection is the strict verdict at the same place
                    assert orc.decode(bytes(t))[1:] == (err, st)


def test_lenient_equals_strict_elsewhere(orc):
    """Lenient differs from strict only on NONCANON verdicts (fuzzed texts, injected errors)."""
    for trial in range(300):
        n = trial * 7
        x = synth.data(n, seed=trial)
        t = orc.encode(x)
        if t.size > 8 and trial % 2:
            pos, bad = synth.corruption(1 + trial % 3, t.size, orc.STANDARD, seed=trial)
            t[pos] = bad
        s = orc.decode(t)
        l = orc.decode(t, lenient=True)
        if s[2] != orc.ST_NONCANON:
            assert s[1:] == l[1:] and s[0].tobytes() == l[0].tobytes()
    # unpadded lenient: the 2/3-char tail's dropped bits may be non-zero (stdlib on re-padded text)
    for g in (b"Zh", b"Zm9", b"QUJDZh", b"QUJDZm9"):
        out, err, st = orc.decode_unpadded(g, lenient=True)
        assert err == -1 and out.tobytes() == binascii.a2b_base64(g + b"=" * (-len(g) % 4), strict_mode=True)
        assert orc.decode_unpadded(g)[2] == orc.ST_NONCANON
    assert orc.decode_ws(b"Z h\n==", lenient=True)[0].tobytes() == b"f"
    assert orc.decode_ws(b"Z h\n==")[1:] == (2, orc.ST_NONCANON)  # original coordinates
    txt = np.frombuffer(b"QUJDZh==Zg==QQ", np.uint8)
    out, off, st, err, olen = orc.decode_batch(txt, np.array([0, 8, 12, 14]), lenient=True)
    assert list(st) == [0, 0, orc.ST_LENGTH] and list(err) == [-1, -1, 0]
    out, off, st, err, olen = orc.decode_batch(txt, np.array([0, 8, 12, 14]))
    assert list(st) == [orc.ST_NONCANON, 0, orc.ST_LENGTH] and list(err) == [5, -1, 0]
